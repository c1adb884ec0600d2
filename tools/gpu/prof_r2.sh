mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"

for spec in "k_lu_apply_strip:SSSSM" "k_qr_apply:TSMQR"; do
  k=${spec%%:*}; kind=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/${k}_${kind}_r2 -f \
    python tools/profile_kinds.py $kind > /dev/null 2>&1
  echo $k=$?
done
