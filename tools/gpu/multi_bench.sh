mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export HG_BENCH_DEVICE=0 HG_DIST_BACKEND=gloo
for spec in "2:cholesky" "4:cholesky" "2:lu" "2:qr"; do
  np=${spec%%:*}; fam=${spec##*:}
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 2951$np \
    bench.py --gpus $np --family $fam --size 8192 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mb_${np}_$fam.log 2>&1
  echo "$np $fam rc=$?"; grep '^{' gpurun_out/mb_${np}_$fam.log | tail -1 | cut -c1-260
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/mb_ref.log 2>&1; echo ref=$?; grep '^{' gpurun_out/mb_ref.log | cut -c1-200
