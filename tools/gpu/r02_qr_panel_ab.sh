#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_qr.py -q -x > $O/qr_ab_tests.log 2>&1; echo "rc=$?" >> $O/qr_ab_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GEQRT TSQRT > $O/qr_ab_tput.jsonl 2>&1
tail -n 3 $O/qr_ab_tests.log; cat $O/qr_ab_tput.jsonl
