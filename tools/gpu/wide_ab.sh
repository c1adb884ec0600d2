mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > gpurun_out/wide_tests.log 2>&1; echo tests=$? >> gpurun_out/wide_tests.log
for w in 1 0; do
  HG_WIDE=$w HG_CONC=8,32 python tools/kind_throughput.py SSSSM GESSM > gpurun_out/kt_wide$w.jsonl 2>&1
done
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_wide.json 2> gpurun_out/bench_lu_wide.err
