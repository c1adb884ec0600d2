mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_tests_all.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_full.log | cut -c1-300
for f in lu qr; do timeout 900 python bench.py --family $f --steps 3 --no-cpu-baseline > gpurun_out/bench_full_$f.log 2>&1; echo $f=$?; tail -1 gpurun_out/bench_full_$f.log | cut -c1-200; done
