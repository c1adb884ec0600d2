mkdir -p gpurun_out
HG_PROF_BATCH=14 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILi128ELi32ELi8ELi32ELi32ELi4 -s 1 -c 1 -o gpurun_out/ssssm_sat -f python tools/prof_batch.py > gpurun_out/ncu_sat.log 2>&1; echo ncu=$?
