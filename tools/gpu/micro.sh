mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
./tools/potrf_micro > gpurun_out/potrf_micro.json 2>&1; echo micro=$?
timeout 600 python tools/kind_throughput.py > gpurun_out/kind_tput.jsonl 2>gpurun_out/kind_tput.err; echo tput=$?
