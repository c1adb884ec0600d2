mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > gpurun_out/strip_tests.log 2>&1; echo tests=$? >> gpurun_out/strip_tests.log
for w in 0 2; do
  HG_WIDE=$w HG_CONC=1,8,32 python tools/kind_throughput.py SSSSM GESSM > gpurun_out/kt_strip$w.jsonl 2>&1
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/kt_strip0.jsonl
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_strip.json 2> gpurun_out/bench_lu_strip.err
