#!/bin/bash
# Session re-entry check on one B200: every GPU test (minus full-size), smoke, bench.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > $O/s5_tests.log 2>&1; echo "rc=$?" >> $O/s5_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/s5_smoke.log 2>&1; echo "rc=$?" >> $O/s5_smoke.log
timeout 900 python bench.py > $O/s5_bench.json 2> $O/s5_bench.err
tail -n 5 $O/s5_tests.log $O/s5_smoke.log; cut -c1-600 $O/s5_bench.json
