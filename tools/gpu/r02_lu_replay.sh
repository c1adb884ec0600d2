#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 900 python tools/lu_replay_check.py 8192 512 128 3 > $O/lu_replay_8192.log 2>&1
timeout 1800 python tools/lu_replay_check.py 32768 1024 128 2 > $O/lu_replay_32768.log 2>&1
tail -3 $O/lu_replay_8192.log $O/lu_replay_32768.log
