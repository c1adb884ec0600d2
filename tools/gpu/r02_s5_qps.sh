#!/bin/bash
# TSQRT panel timeline before/after the norm downdating. The 'old' build needs the pre-change kernel, e.g.
#   mkdir -p tools/ab && git show 4392b43:paper_1402_6601_b200/csrc/tiles_qr.cu > tools/ab/tiles_qr_old.cu &&
#   sed 's#../paper_1402_6601_b200/csrc/tiles_qr.cu#tiles_qr_old.cu#' tools/qr_panel_stamps.cu > tools/ab/qps_old.cu
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHG_PANEL_STAMPS -I paper_1402_6601_b200/csrc -I include"
nvcc $F tools/qr_panel_stamps.cu -o /tmp/qps_new > $O/qps_build.log 2>&1
nvcc $F -I tools/ab tools/ab/qps_old.cu -o /tmp/qps_old >> $O/qps_build.log 2>&1
for i in 1 2; do /tmp/qps_new t; /tmp/qps_old t; done > $O/qps.jsonl 2>&1
tail -3 $O/qps_build.log; cut -c1-400 $O/qps.jsonl
