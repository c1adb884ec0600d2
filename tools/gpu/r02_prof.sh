#!/bin/bash
# Saturated-mix profiles of the LU/QR trailing updates and the panel kernels (ncu range replay:
# 32 independent tasks on 32 streams measured as one workload), plus the panel kernel alone.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
for K in SSSSM TSMQR TSTRF; do
  HG_PROF_RANGE=1 HG_CONC=32 timeout 900 ncu --replay-mode range --profile-from-start off --set full \
    --clock-control none -f -o $O/r02_range_$K python tools/kind_throughput.py $K > $O/r02_range_$K.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_panel_sp -s 2 -c 1 -f \
  -o $O/r02_lu_panel_sp python tools/kind_throughput.py TSTRF > $O/r02_lu_panel_sp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_apply_strip -s 40 -c 1 -f \
  -o $O/r02_lu_strip python tools/kind_throughput.py SSSSM > $O/r02_lu_strip.log 2>&1
ls -la $O/*.ncu-rep
