python -c "import __graft_entry__ as g; g.build()"
echo "== default"; timeout 300 python tools/debug_lu_k2.py lu
echo "== apply16"; HG_LU_APPLY=16 timeout 300 python tools/debug_lu_k2.py lu
echo "== apply16 prio0"; HG_PRIORITY_LEVELS=0 HG_LU_APPLY=16 timeout 300 python tools/debug_lu_k2.py lu
echo "== qr default"; timeout 300 python tools/debug_lu_k2.py qr
echo "== chol default"; timeout 300 python tools/debug_lu_k2.py cholesky
