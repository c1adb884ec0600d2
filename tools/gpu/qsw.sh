mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qr.py -x -q > gpurun_out/qsw_tests.log 2>&1; echo tests=$? >> gpurun_out/qsw_tests.log
HG_CONC=1,32 python tools/kind_throughput.py TSMQR UNMQR TSQRT > gpurun_out/kt_qsw.jsonl 2>&1
python bench.py --family qr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qr_qsw.json 2> gpurun_out/bench_qr_qsw.err
