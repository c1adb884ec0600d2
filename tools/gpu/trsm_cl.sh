mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cholesky.py tests/test_gpu_edges.py tests/test_gpu_virtual_nodes.py tests/test_gpu_multirank.py -x -q > gpurun_out/tc_tests.log 2>&1; echo tests=$? >> gpurun_out/tc_tests.log
HG_CONC=1,32 timeout 300 python tools/kind_throughput.py TRSM > gpurun_out/kt_tc.jsonl 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_tc.json 2> /dev/null
for i in 1 2; do timeout 300 python tools/c5probe.py 65536 > gpurun_out/c5_tc_$i.json 2> gpurun_out/c5_tc_$i.err; echo c5_$i=$? >> gpurun_out/tc_tests.log; done
