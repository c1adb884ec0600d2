python -c "import __graft_entry__ as g; g.build()"
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline $BARGS 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['value']), round(d['ms_per_step'],1))"; }
BARGS="--family lu"; run lu_s32 X=1; run lu_s64 HG_LU_APPLY=64
BARGS="--family qr"; run qr_s32 X=1; run qr_s64 HG_QR_APPLY=64
HG_CONC=1,32 HG_LU_APPLY=64 HG_QR_APPLY=64 timeout 300 python tools/kind_throughput.py SSSSM TSMQR
