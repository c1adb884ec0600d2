#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_online.py -q -x > $O/v_mr.log 2>&1; echo "rc=$?" >> $O/v_mr.log
HG_PARITY_OUT=$O/r02_parity_lu.jsonl timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -k "lu" > $O/v_full_lu.log 2>&1; echo "rc=$?" >> $O/v_full_lu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_panel_sp -c 1 -f \
  -o $O/r02_lu_panel_sp python tools/profile_kinds.py TSTRF > $O/r02_lu_panel_sp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qr_panel -c 1 -f \
  -o $O/r02_qr_panel python tools/profile_kinds.py TSQRT > $O/r02_qr_panel.log 2>&1
tail -n 3 $O/v_mr.log $O/v_full_lu.log 2>/dev/null; cat $O/r02_parity_lu.jsonl
