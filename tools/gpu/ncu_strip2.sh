mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for spec in "k_lu_apply_strip:SSSSM" "k_qr_apply:TSMQR" "k_lu_panel_sp:TSTRF"; do
  k=${spec%%:*}; kind=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 2 -k regex:$k -c 1 -o gpurun_out/${k}_${kind}2 -f \
    python tools/profile_kinds.py $kind > /dev/null 2>&1
  echo $k=$?
done
