#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 900 python bench.py > $O/b8_bench.json 2> $O/b8_bench.err
python -c "
import json;d=json.load(open('$O/b8_bench.json'));print(d['value'], json.dumps(d['e2e']), d['one_shot']['registered']['register_ms'])"
