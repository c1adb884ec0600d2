mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cholesky.py -x -q > gpurun_out/g4_tests.log 2>&1; echo tests=$? >> gpurun_out/g4_tests.log
HG_GEMM_STAGES=4 HG_GEMM_STAGES=4 python tools/kind_throughput.py GEMM SYRK > gpurun_out/kt_g4.jsonl 2>&1
python bench.py > gpurun_out/bench_c2_g3.json 2> /dev/null
HG_GEMM_STAGES=4 python bench.py > gpurun_out/bench_c2_g4.json 2> /dev/null
python bench.py > gpurun_out/bench_c2_g3b.json 2> /dev/null
