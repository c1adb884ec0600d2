mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/nd2_tests.log 2>&1; echo tests=$? >> gpurun_out/nd2_tests.log
HG_CONC=1,8,32 python tools/kind_throughput.py GEMM SYRK TRSM TSMQR UNMQR > gpurun_out/kt_nd2.jsonl 2>&1
python bench.py > gpurun_out/bench_c2_nd2.json 2> gpurun_out/bench_c2_nd2.err
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_nd2.json 2> gpurun_out/bench_lu_nd2.err
python bench.py --family qr --steps 3 --warmup 3 > gpurun_out/bench_qr_nd2.json 2> gpurun_out/bench_qr_nd2.err
