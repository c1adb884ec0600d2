#!/bin/bash
cd "$GRAFT_REPO_ROOT"
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1402_6601_b200/csrc -I include"
nvcc $F -DHG_PANEL_STAMPS tools/ssssm_ab.cu -o /tmp/abs 2>/dev/null; /tmp/abs; /tmp/abs q
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_qr.py -q -x 2>&1 | tail -n 2
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GESSM SSSSM UNMQR TSMQR GETRF_INC TSTRF GEQRT TSQRT 2>&1 | cut -c1-200
