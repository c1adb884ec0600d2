#!/bin/bash
# re-check after the VLoader mask fix + balanced top' solve: LU/QR/virtual-node/tile-shape tests, kinds, bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py tests/test_gpu_virtual_nodes.py tests/test_gpu_tile_shapes.py tests/test_gpu_multirank.py tests/test_gpu_online.py -q -x > $O/fx_tests.log 2>&1; echo "rc=$?" >> $O/fx_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py SSSSM GESSM TSMQR UNMQR > $O/fx_kinds.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/fx_bench.json 2> $O/fx_bench.err
tail -n 8 $O/fx_tests.log; cat $O/fx_kinds.jsonl | cut -c1-200; python -c "
import json;d=json.load(open('$O/fx_bench.json'));print(d['value'], json.dumps(d['families_k1'])[:700])"
