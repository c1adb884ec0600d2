#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_multirank.py -q -x > $O/lu_ab_tests.log 2>&1; echo "rc=$?" >> $O/lu_ab_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GETRF_INC TSTRF SSSSM > $O/lu_ab_tput.jsonl 2>&1
tail -n 3 $O/lu_ab_tests.log; cat $O/lu_ab_tput.jsonl
