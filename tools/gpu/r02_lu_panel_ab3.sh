#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHG_PANEL_STAMPS -I paper_1402_6601_b200/csrc -I include tools/panel_stamps.cu -o /tmp/ps && /tmp/ps t > $O/stamps3_t.json && /tmp/ps g > $O/stamps3_g.json
timeout 600 python -m pytest tests/test_gpu_lu.py -q -x > $O/lu_ab3_tests.log 2>&1; echo "rc=$?" >> $O/lu_ab3_tests.log
HG_CONC=1,32 timeout 600 python tools/kind_throughput.py GETRF_INC TSTRF > $O/lu_ab3_tput.jsonl 2>&1
tail -n 3 $O/lu_ab3_tests.log; cat $O/lu_ab3_tput.jsonl; cut -c1-400 $O/stamps3_t.json $O/stamps3_g.json
