#!/bin/bash
# Session-5 final validation (after TMA + TSQRT norm downdating): all GPU tests incl. full-size parity,
# smoke, all-kind throughput on fresh operands, bench (ours + reference arm with baseline/_ref),
# LU launch list (kernel shares) and one full ncu capture of the TSQRT panel.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > $O/g6_tests.log 2>&1; echo "rc=$?" >> $O/g6_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/g6_smoke.log 2>&1; echo "rc=$?" >> $O/g6_smoke.log
HG_CONC=1,32 timeout 1200 python tools/kind_throughput.py > $O/g6_kinds.jsonl 2>&1
timeout 900 python bench.py > $O/g6_bench.json 2> $O/g6_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/g6_ref.json 2> $O/g6_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 25000 --csv --log-file $O/g6_launches_lu.csv python bench.py --family lu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-extra-families --no-one-shot > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qr_panel -s 0 -c 1 -f -o $O/g6_qr_panel python tools/profile_kinds.py TSQRT > /dev/null 2>&1
HG_PARITY_OUT=$O/g6_parity.jsonl timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -s > $O/g6_fullsize.log 2>&1; echo "rc=$?" >> $O/g6_fullsize.log
tail -n 3 $O/g6_tests.log $O/g6_fullsize.log $O/g6_smoke.log 2>/dev/null; cut -c1-160 $O/g6_parity.jsonl; cut -c1-160 $O/g6_kinds.jsonl
