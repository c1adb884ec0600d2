mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py -x -q > gpurun_out/tri_tests.log 2>&1; echo tests=$? >> gpurun_out/tri_tests.log
HG_CONC=1,32 python tools/kind_throughput.py TSMQR UNMQR SSSSM GESSM > gpurun_out/kt_tri.jsonl 2>&1
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_tri.json 2> gpurun_out/bench_lu_tri.err
python bench.py --family qr --steps 3 --warmup 3 > gpurun_out/bench_qr_tri.json 2> gpurun_out/bench_qr_tri.err
