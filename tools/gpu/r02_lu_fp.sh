#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHG_PANEL_STAMPS -I paper_1402_6601_b200/csrc -I include tools/panel_stamps.cu -o /tmp/ps && /tmp/ps t | cut -c1-330
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_tile_shapes.py tests/test_gpu_virtual_nodes.py -q -x 2>&1 | tail -n 2
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GETRF_INC TSTRF SSSSM GESSM 2>&1 | cut -c1-200
python bench.py --family lu > $O/bench_lu.json 2> $O/bench_lu.err; python -c "
import json; d=json.loads(open('$O/bench_lu.json').read().strip().splitlines()[-1]); print('LU C3 k=1', d['value'], d['ms_per_step'])"
