#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_online.py tests/test_capi.py -q -x > $O/online.log 2>&1; echo "online rc=$?" >> $O/online.log
timeout 2400 python tools/lu_sensitivity.py 32768 1024 128 2 > $O/lu_sens_32768.json 2> $O/lu_sens_32768.err
for K in SSSSM TSMQR; do
  HG_PROF_RANGE=1 HG_CONC=32 timeout 900 ncu --replay-mode range --set full \
    --clock-control none -f -o $O/r02_range_$K python tools/kind_throughput.py $K > $O/r02_range_$K.log 2>&1
done
tail -n 3 $O/online.log; cat $O/lu_sens_32768.json; tail -n 3 $O/lu_sens_32768.err; ls $O
