# one full ncu capture (source-level) of each critical-path panel kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for spec in "k_lu_panel:GETRF_INC" "k_qr_panel:GEQRT" "k_potrf_cluster:POTRF"; do
  k=${spec%%:*}; kind=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/$k -f \
    python tools/profile_kinds.py $kind > gpurun_out/ncu_$k.log 2>&1
  echo $k=$?
done
