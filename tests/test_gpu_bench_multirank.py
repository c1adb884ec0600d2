"""bench.py's N > 1 path end to end (torchrun, one process per GPU node, CUDA IPC
pools, device flags, step fences, max-over-ranks timing, executed-bytes check).
Needs two GPUs: ranks whose kernels wait on one another must not share one GPU
as separate processes (see tests/test_gpu_multirank.py); on a 1-GPU box the
N > 1 host logic is covered on the CPU (tests/test_multirank.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("family", ["cholesky", "lu"])
def test_bench_two_ranks(family):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("one process per GPU: needs 2 GPUs (ranks that wait on one another must not share a GPU)")
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--family", family, "--size", "4096", "--nb", "512", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 prints one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["nvlink_bytes"]["dada"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
