#!/bin/bash
# Session-5 validation on one B200 after the LU/QR push + warp-private update streams: every GPU test
# (incl. full-size parity), smoke, all-kind throughput (cost tables), bench (ours + reference arm),
# the bench's ncu launch list and full captures of the two rebuilt trailing-update kernels.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > $O/f5_tests.log 2>&1; echo "rc=$?" >> $O/f5_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/f5_smoke.log 2>&1; echo "rc=$?" >> $O/f5_smoke.log
HG_CONC=1,32 timeout 900 python tools/kind_throughput.py > $O/f5_kinds.jsonl 2>&1
timeout 900 python bench.py > $O/f5_bench.json 2> $O/f5_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/f5_ref.json 2> $O/f5_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/f5_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_apply_strip -s 60 -c 1 -f -o $O/f5_lu_strip python tools/kind_throughput.py SSSSM > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qr_apply -s 60 -c 1 -f -o $O/f5_qr_apply python tools/kind_throughput.py TSMQR > /dev/null 2>&1
HG_PARITY_OUT=$O/f5_parity.jsonl timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -s > $O/f5_fullsize.log 2>&1; echo "rc=$?" >> $O/f5_fullsize.log
tail -n 3 $O/f5_tests.log $O/f5_fullsize.log $O/f5_smoke.log 2>/dev/null; cut -c1-200 $O/f5_parity.jsonl; cut -c1-200 $O/f5_kinds.jsonl
