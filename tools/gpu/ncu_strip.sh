mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for spec in "k_lu_apply_strip:SSSSM" "k_qr_apply:TSMQR"; do
  k=${spec%%:*}; kind=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/${k}_$kind -f \
    python tools/profile_kinds.py $kind > gpurun_out/ncu_${k}.log 2>&1
  echo $k=$?
done
