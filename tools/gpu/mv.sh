mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > gpurun_out/mv_tests.log 2>&1; echo tests=$? >> gpurun_out/mv_tests.log
for b in 1 14; do HG_PROF_BATCH=$b python tools/prof_batch.py; done > gpurun_out/prof_batch_mv.txt 2>&1
HG_CONC=1,32 python tools/kind_throughput.py SSSSM GESSM > gpurun_out/kt_mv.jsonl 2>&1
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_mv.json 2> gpurun_out/bench_lu_mv.err
