mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
./tools/potrf_micro > gpurun_out/potrf_micro3.json 2>&1; echo micro=$?; cat gpurun_out/potrf_micro3.json
timeout 600 python -m pytest tests/test_gpu_cholesky.py tests/test_gpu_multirank.py -x -q > gpurun_out/gpu_tests_chol.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests_chol.log
timeout 300 python tools/kind_throughput.py POTRF; echo tput=$?
timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_chol4.log 2>&1; echo chol=$?
tail -1 gpurun_out/bench_chol4.log | cut -c1-200
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_qr_panel -c 1 -o gpurun_out/k_qr_panel_hi -f python tools/profile_kinds.py GEQRT > gpurun_out/ncu_qr_hi.log 2>&1; echo ncu=$?
