#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
for cfg in "8192 512 1 1 1" "8192 512 1 0 1" "8192 512 3 1 0" "4096 512 1 1 1"; do
  timeout 600 python tools/debug_multirank_lu.py $cfg >> $O/dbg_mr.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_lu.py -q -x >> $O/dbg_mr.log 2>&1
# saturated profiles of the LU/QR trailing updates and the panel kernels
for K in SSSSM TSMQR; do
  HG_PROF_RANGE=1 HG_CONC=32 timeout 900 ncu --replay-mode range --profile-from-start off --set full \
    --clock-control none -f -o $O/r02_range_$K python tools/kind_throughput.py $K > $O/r02_range_$K.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_apply_strip -s 40 -c 1 -f \
  -o $O/r02_lu_strip python tools/profile_kinds.py SSSSM > $O/r02_lu_strip.log 2>&1
cat $O/dbg_mr.log | grep -v "^\.\|passed" | head -60
