mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
echo "== default"; timeout 300 python tools/debug_lu_k2.py lu
echo "== apply16"; HG_LU_APPLY=16 timeout 300 python tools/debug_lu_k2.py lu
echo "== qr"; timeout 300 python tools/debug_lu_k2.py qr
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_all.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests_all.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline $BARGS > gpurun_out/ab2_$tag.log 2>&1; echo $tag=$?; }
BARGS="--family lu"
run lu_s32
run lu_s64 HG_LU_APPLY=64
BARGS="--family qr"
run qr_s32
BARGS=""
run chol
