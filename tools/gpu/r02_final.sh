#!/bin/bash
# Round-2 final validation on one B200: every GPU test (incl. full-size parity), smoke, bench (ours +
# reference arm), ncu launch list of the bench and full captures of the rebuilt kernels.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > $O/final_tests.log 2>&1; echo "rc=$?" >> $O/final_tests.log
HG_PARITY_OUT=$O/final_parity.jsonl timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -s > $O/final_fullsize.log 2>&1; echo "rc=$?" >> $O/final_fullsize.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; echo "rc=$?" >> $O/final_smoke.log
timeout 900 python bench.py > $O/final_bench.json 2> $O/final_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/final_ref.json 2> $O/final_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/final_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_apply_strip -s 60 -c 1 -f -o $O/final_lu_strip python tools/kind_throughput.py SSSSM > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_panel_sp -c 1 -f -o $O/final_lu_panel python tools/profile_kinds.py TSTRF > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qr_panel -c 1 -f -o $O/final_qr_panel python tools/profile_kinds.py TSQRT > /dev/null 2>&1
tail -n 3 $O/final_tests.log $O/final_fullsize.log $O/final_smoke.log 2>/dev/null; cat $O/final_parity.jsonl | cut -c1-200
