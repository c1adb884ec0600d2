#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHG_PANEL_STAMPS -I paper_1402_6601_b200/csrc -I include tools/qr_panel_stamps.cu -o /tmp/qps && /tmp/qps g | cut -c1-330
timeout 900 python -m pytest tests/test_gpu_qr.py -q -x 2>&1 | tail -n 2
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GEQRT TSQRT 2>&1
python bench.py --family qr > $O/bench_qr.json 2> $O/bench_qr.err; python -c "
import json; d=json.loads(open('$O/bench_qr.json').read().strip().splitlines()[-1]); print('QR C4 k=1', d['value'], d['ms_per_step'])"
