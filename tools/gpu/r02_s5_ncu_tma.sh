#!/bin/bash
# ncu of the TMA-staged LU strip kernel (SSSSM, one launch, fresh operands) + SASS evidence of UTMALDG
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lu_apply_strip -s 60 -c 1 -f -o $O/n10_lu_strip python tools/kind_throughput.py SSSSM > $O/n10.log 2>&1
cuobjdump -sass -fun '_ZN2hg16k_lu_apply_stripINS_7GemmCfgILi128ELi32ELi8ELi32ELi32ELi4ELb0EEELb1ES2_EEvNS_13LuApplyParamsE' paper_1402_6601_b200/libhetgpu.so 2>/dev/null | grep -c UTMALDG > $O/n10_sass.txt
tail -2 $O/n10.log; cat $O/n10_sass.txt
