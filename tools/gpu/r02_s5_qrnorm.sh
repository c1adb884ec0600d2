#!/bin/bash
# TSQRT column-norm downdating (one message exchange per column instead of two): QR tests, panel kinds, bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_qr.py tests/test_gpu_virtual_nodes.py tests/test_gpu_tile_shapes.py -q > $O/qn_tests.log 2>&1; echo "rc=$?" >> $O/qn_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py TSQRT GEQRT TSMQR > $O/qn_kinds.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-one-shot > $O/qn_bench.json 2> $O/qn_bench.err
tail -n 4 $O/qn_tests.log; cut -c1-200 $O/qn_kinds.jsonl; python -c "
import json;d=json.load(open('$O/qn_bench.json'));print(d['value'], json.dumps(d['families_k1'])[:600])"
