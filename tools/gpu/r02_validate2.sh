#!/bin/bash
# Round-2 re-entry validation on one B200: GPU tests (minus full-size), bench, full-size LU/QR element-wise parity.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > $O/r02v2_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r02v2_gpu_tests.log
timeout 900 python bench.py > $O/r02v2_bench.json 2> $O/r02v2_bench.err
HG_PARITY_OUT=$O/r02v2_parity_full.jsonl timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -k "lu or qr" > $O/r02v2_fullsize.log 2>&1; echo "fullsize rc=$?" >> $O/r02v2_fullsize.log
tail -3 $O/r02v2_gpu_tests.log; tail -3 $O/r02v2_fullsize.log; cat $O/r02v2_parity_full.jsonl
