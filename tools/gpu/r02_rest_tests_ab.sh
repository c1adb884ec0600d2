#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
bash tools/gpu/r02_ssssm_ab.sh > $O/ssssm_ab.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > $O/full_tests2.log 2>&1; echo "rc=$?" >> $O/full_tests2.log
tail -n 5 $O/full_tests2.log; cat $O/ssssm_ab.log
