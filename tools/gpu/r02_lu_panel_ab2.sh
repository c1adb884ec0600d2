#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_lu.py -q -x > $O/lu_ab2_tests.log 2>&1; echo "rc=$?" >> $O/lu_ab2_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GETRF_INC TSTRF > $O/lu_ab2_tput.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_panel_sp -c 1 -f \
  -o $O/r02_lu_panel_sp2 python tools/profile_kinds.py TSTRF > $O/r02_lu_panel_sp2.log 2>&1
tail -n 3 $O/lu_ab2_tests.log; cat $O/lu_ab2_tput.jsonl
