#!/bin/bash
# LU strip kernel with the pristine top rows staged by a tensor-map TMA box: LU tests, SSSSM/GESSM throughput, bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lu.py tests/test_gpu_virtual_nodes.py tests/test_gpu_tile_shapes.py tests/test_gpu_online.py tests/test_gpu_edges.py -q > $O/tm_tests.log 2>&1; echo "rc=$?" >> $O/tm_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py SSSSM GESSM TSTRF GETRF_INC > $O/tm_kinds.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/tm_bench.json 2> $O/tm_bench.err
cuobjdump -sass paper_1402_6601_b200/libhetgpu.so | grep -c UTMALDG > $O/tm_sass.txt
tail -n 4 $O/tm_tests.log; cut -c1-200 $O/tm_kinds.jsonl; python -c "
import json;d=json.load(open('$O/tm_bench.json'));print(d['value'], json.dumps(d['families_k1'])[:400])"
