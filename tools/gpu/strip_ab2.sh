mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py -x -q > gpurun_out/strip2_tests.log 2>&1; echo tests=$? >> gpurun_out/strip2_tests.log
HG_CONC=1,8,32,64 python tools/kind_throughput.py TSMQR UNMQR SSSSM > gpurun_out/kt_strip2_new.jsonl 2>&1
HG_QR_APPLY=32 HG_CONC=1,8,32 python tools/kind_throughput.py TSMQR UNMQR > gpurun_out/kt_strip2_old.jsonl 2>&1
python bench.py --family qr --steps 3 --warmup 3 > gpurun_out/bench_qr_strip.json 2> gpurun_out/bench_qr_strip.err
python bench.py --family lu --steps 3 --warmup 3 > gpurun_out/bench_lu_strip.json 2> gpurun_out/bench_lu_strip.err
