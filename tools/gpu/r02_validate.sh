#!/bin/bash
# Round-2 validation on one B200: GPU tests (minus the long full-size file), bench (ours + reference arm),
# full-size element-wise parity, CPU-column calibration of the cost tables on this host.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > $O/r02_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r02_gpu_tests.log
timeout 900 python bench.py > $O/r02_bench1.json 2> $O/r02_bench1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/r02_ref1.json 2> $O/r02_ref1.err
HG_PARITY_OUT=$O/r02_parity_full2.jsonl timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > $O/r02_fullsize2.log 2>&1; echo "fullsize rc=$?" >> $O/r02_fullsize2.log
mkdir -p $O/timings && cp timings/*.csv $O/timings/ && timeout 900 python tools/calibrate.py --cpu-only $O/timings/b200_nb1024_ib128.csv $O/timings/b200_nb1024_ib128_tput.csv > $O/r02_cpu_column.log 2>&1
tail -3 $O/r02_gpu_tests.log; tail -2 $O/r02_fullsize2.log
