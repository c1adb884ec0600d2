#!/bin/bash
# phase breakdown (CTA 0 stamps of one task among 32 concurrent) of SSSSM / TSMQR with this session's kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1402_6601_b200/csrc -I include"
nvcc $F -DHG_PANEL_STAMPS tools/ssssm_ab.cu -o /tmp/abs > $O/st_build.log 2>&1 && nvcc $F tools/ssssm_ab.cu -o /tmp/ab0 >> $O/st_build.log 2>&1
for k in s q; do for i in 1 2; do /tmp/abs $k; /tmp/ab0 $k; done; done > $O/st_stamps.jsonl 2>&1
cat $O/st_build.log | tail -3; cat $O/st_stamps.jsonl
