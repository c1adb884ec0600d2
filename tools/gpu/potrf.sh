mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
./tools/potrf_micro > gpurun_out/potrf_micro2.json 2>&1; echo micro=$?
timeout 600 python -m pytest tests/test_gpu_cholesky.py -x -q > gpurun_out/gpu_tests_chol.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests_chol.log
timeout 300 python tools/kind_throughput.py POTRF TRSM SYRK GEMM SSSSM GESSM TSMQR UNMQR > gpurun_out/kind_tput.jsonl 2>gpurun_out/kind_tput.err; echo tput=$?
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_chol3.log 2>&1; echo chol=$?
tail -1 gpurun_out/bench_chol3.log | cut -c1-300
