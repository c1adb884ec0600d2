#!/bin/bash
cd "$GRAFT_REPO_ROOT"
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1402_6601_b200/csrc -I include"
nvcc $F tools/ssssm_ab.cu -o /tmp/ab0 && nvcc $F -DHG_EXP_RED_AS_STORE tools/ssssm_ab.cu -o /tmp/ab1 && nvcc $F -DHG_EXP_NO_MOVES tools/ssssm_ab.cu -o /tmp/ab2 && nvcc $F -DHG_EXP_NO_MOVES -DHG_EXP_RED_AS_STORE tools/ssssm_ab.cu -o /tmp/ab3
for i in 0 1 2 3; do echo "variant $i: $(/tmp/ab$i)"; done
