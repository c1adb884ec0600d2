mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_qr.py -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed|error" | head -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qrsp_launches.csv python tools/profile_kinds.py GEQRT TSQRT > /dev/null 2>&1
python3 - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/qrsp_launches.csv')) if len(r)>10]
h=rows[0]; i={k:n for n,k in enumerate(h)}
for r in rows[1:]:
    if r[i['Metric Name']]=='gpu__time_duration.sum' and 'hg::' in r[i['Kernel Name']]:
        print(r[i['Kernel Name']].split('(')[0][:40], r[i['Grid Size']], float(r[i['Metric Value']])/1000)
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_qr_panel_sp -c 1 -o gpurun_out/k_qr_panel_sp -f python tools/profile_kinds.py GEQRT > /dev/null 2>&1; echo ncu=$?
