mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo ncu=$?
timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_quick.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_quick.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['roofline']))"
