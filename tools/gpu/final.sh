mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --family lu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_lu.json 2> /dev/null
python bench.py --family qr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_qr.json 2> /dev/null
