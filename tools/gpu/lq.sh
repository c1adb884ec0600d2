mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_lu.py -x -q > gpurun_out/gpu_tests_lq.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests_lq.log
HG_CONC=1,8,32 timeout 300 python tools/kind_throughput.py SSSSM GESSM TSMQR UNMQR > gpurun_out/kind_tput2.jsonl 2>gpurun_out/kind_tput2.err; echo tput=$?
cat gpurun_out/kind_tput2.jsonl
for fam in lu qr; do timeout 600 python bench.py --family $fam --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${fam}4.log 2>&1; echo $fam=$?; tail -1 gpurun_out/bench_${fam}4.log | cut -c1-250; done
