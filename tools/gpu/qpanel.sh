mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_edges.py -x -q > gpurun_out/qp_tests.log 2>&1; echo tests=$? >> gpurun_out/qp_tests.log
HG_CONC=1,32 python tools/kind_throughput.py GEQRT TSQRT > gpurun_out/kt_qp.jsonl 2>&1
python bench.py --family qr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qr_qp.json 2> /dev/null
