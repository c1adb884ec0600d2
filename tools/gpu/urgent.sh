mkdir -p gpurun_out
HG_URGENT=1 timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py -x -q > gpurun_out/urg_tests.log 2>&1; echo tests=$? >> gpurun_out/urg_tests.log
for fam in lu qr; do
  for u in 1 0; do HG_URGENT=$u timeout 300 python bench.py --family $fam --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${fam}_urg$u.json 2>/dev/null; done
done
