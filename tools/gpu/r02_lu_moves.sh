#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1402_6601_b200/csrc -I include"
nvcc $F tools/ssssm_ab.cu -o /tmp/ab0 2>/dev/null && echo "ssssm_ab: $(/tmp/ab0)"
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_virtual_nodes.py -q -x 2>&1 | tail -n 3
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GETRF_INC GESSM TSTRF SSSSM 2>&1
