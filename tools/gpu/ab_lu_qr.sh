mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_lu.py -x -q > gpurun_out/gpu_tests_ab.log 2>&1; echo tests=$?
HG_LU_APPLY=16 timeout 600 python -m pytest tests/test_gpu_lu.py -x -q > gpurun_out/gpu_tests_ab16.log 2>&1; echo tests16=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kinds_launches4.csv \
  python tools/profile_kinds.py GETRF_INC GESSM TSTRF SSSSM GEQRT UNMQR TSQRT TSMQR > gpurun_out/kinds4.log 2>&1; echo ncu=$?
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline $BARGS > gpurun_out/ab_$tag.log 2>&1; echo $tag=$?; }
BARGS="--family lu"
run lu_sp_s32
HG_X=1 run lu_reg_s32 HG_LU_PANEL=reg
run lu_sp_s16 HG_LU_APPLY=16
BARGS="--family qr"
run qr_s32
run qr_s64 HG_QR_APPLY=64
run qr_s16 HG_QR_APPLY=16
