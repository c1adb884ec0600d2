mkdir -p gpurun_out timings
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python tools/calibrate.py --nb 1024 --ib 128 --out gpurun_out/b200_nb1024_ib128.csv > gpurun_out/calib.log 2>&1; echo calib=$?
cp gpurun_out/b200_nb1024_ib128.csv timings/ 2>/dev/null
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo ncu=$?
