mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_lu.py -x -q > gpurun_out/gpu_tests_lu3.log 2>&1; echo tests=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kinds_launches3.csv \
  python tools/profile_kinds.py GETRF_INC TSTRF SSSSM TSMQR > gpurun_out/kinds3.log 2>&1; echo ncu=$?
for spec in "k_qr_apply_cl:TSMQR" "k_lu_apply_cl:SSSSM" "k_lu_panel_sp:GETRF_INC"; do
  k=${spec%%:*}; kind=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/$k -f \
    python tools/profile_kinds.py $kind > gpurun_out/ncu_$k.log 2>&1
  echo $k=$?
done
