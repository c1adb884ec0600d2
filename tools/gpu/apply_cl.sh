mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
HG_PRIORITY_LEVELS=0 timeout 300 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/mr_p0.log 2>&1; echo mr0=$?
HG_PRIORITY_LEVELS=6 timeout 300 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/mr_p6.log 2>&1; echo mr6=$?
timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_lu.py -x -q > gpurun_out/gpu_tests_lq.log 2>&1; echo tests=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kinds_launches2.csv \
  python tools/profile_kinds.py GETRF_INC GESSM TSTRF SSSSM GEQRT UNMQR TSQRT TSMQR > gpurun_out/kinds2.log 2>&1; echo ncu=$?
timeout 900 python bench.py --family lu --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_lu2.log 2>&1; echo lu=$?
timeout 900 python bench.py --family qr --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_qr2.log 2>&1; echo qr=$?
