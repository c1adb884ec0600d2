#!/bin/bash
# last check of HEAD (regenerated cost tables): GPU tests (minus full-size), smoke, bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > $O/h7_tests.log 2>&1; echo "rc=$?" >> $O/h7_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/h7_smoke.log 2>&1; echo "rc=$?" >> $O/h7_smoke.log
timeout 900 python bench.py > $O/h7_bench.json 2> $O/h7_bench.err
tail -n 2 $O/h7_tests.log $O/h7_smoke.log; python -c "
import json;d=json.load(open('$O/h7_bench.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], json.dumps(d['families_k1'])[:500])"
