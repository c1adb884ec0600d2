# launch lists of every tile kind (one task each, 2 reps), then LU/QR step benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kinds_launches.csv \
  python tools/profile_kinds.py POTRF TRSM SYRK GEMM GETRF_INC GESSM TSTRF SSSSM GEQRT UNMQR TSQRT TSMQR > gpurun_out/kinds.log 2>&1
echo ncu=$?
timeout 900 python bench.py --family lu --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lu.log 2>&1; echo lu=$?
timeout 900 python bench.py --family qr --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qr.log 2>&1; echo qr=$?
