mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py -x -q > gpurun_out/red_tests.log 2>&1; echo tests=$? >> gpurun_out/red_tests.log
for r in 1 0; do
  HG_RED=$r HG_CONC=8,32 python tools/kind_throughput.py SSSSM TSMQR GESSM UNMQR > gpurun_out/kt_red$r.jsonl 2>&1
done
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_red1.json 2> gpurun_out/bench_lu_red1.err
python bench.py --family qr --steps 3 --warmup 3 > gpurun_out/bench_qr_red1.json 2> gpurun_out/bench_qr_red1.err
