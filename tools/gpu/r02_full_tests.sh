#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > $O/full_tests.log 2>&1; echo "rc=$?" >> $O/full_tests.log
HG_CONC=1,32 timeout 900 python tools/kind_throughput.py > $O/kinds_all.jsonl 2>&1
tail -n 3 $O/full_tests.log; cat $O/kinds_all.jsonl
