mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_gemm_nt -s 1 -c 1 -o gpurun_out/gemm_prof_r01b -f python tools/profile_kinds.py GEMM > gpurun_out/ncu_gemm.log 2>&1; echo ncu2=$?
