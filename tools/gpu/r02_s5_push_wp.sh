#!/bin/bash
# LU/QR producer-push + warp-private update streams: parity tests, kind throughput, bench.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py tests/test_gpu_virtual_nodes.py tests/test_gpu_tile_shapes.py tests/test_gpu_multirank.py tests/test_gpu_bench_multirank.py -q > $O/pw_tests.log 2>&1; echo "rc=$?" >> $O/pw_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py SSSSM GESSM TSMQR UNMQR > $O/pw_kinds.jsonl 2>&1
timeout 900 python bench.py > $O/pw_bench.json 2> $O/pw_bench.err
tail -n 8 $O/pw_tests.log; cat $O/pw_kinds.jsonl | cut -c1-300; python -c "
import json;d=json.load(open('$O/pw_bench.json'));print(d['value'], json.dumps(d['families_k1'])[:600])"
