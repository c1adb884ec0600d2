mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for pl in 0 6; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --priority-levels $pl > gpurun_out/prio_chol_$pl.log 2>&1; echo chol$pl=$?
  timeout 600 python bench.py --family qr --steps 2 --no-e2e --no-cpu-baseline --priority-levels $pl > gpurun_out/prio_qr_$pl.log 2>&1; echo qr$pl=$?
done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
