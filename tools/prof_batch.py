"""One saturated SSSSM launch for ncu: HG_PROF_BATCH operand sets in one grid.
    HG_PROF_BATCH=14 python tools/prof_batch.py   (sets the stride itself)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

nb, ib = 1024, 128
side = ib * nb + nb
T = nb * nb + side
B = int(os.environ.get("HG_PROF_BATCH", "14"))
os.environ["HG_PROF_STRIDE"] = str(3 * T)
import paper_1402_6601_b200 as H  # noqa: E402
from paper_1402_6601_b200 import _native  # noqa: E402

L = _native.lib()
status = torch.zeros(1, dtype=torch.int32, device="cuda")
rng = np.random.default_rng(0)
buf = torch.zeros(B * 3 * T, dtype=torch.float64, device="cuda")
for i in range(3):
    a = rng.uniform(-0.5, 0.5, (nb, nb))
    buf[i * T: i * T + nb * nb] = torch.from_numpy(np.asfortranarray(a).ravel(order="F")).cuda()
ptr = lambda i: buf.data_ptr() + 8 * i * T
def run(kind, idx):
    p = (C.c_void_p * len(idx))(*[ptr(i) for i in idx])
    _native.check(L.hg_tile_run(H.ALL_KINDS.index(kind), 0, None, p, len(idx), nb, ib,
                                C.c_void_p(status.data_ptr())), kind)

run("GETRF_INC", [0])
run("TSTRF", [0, 1])
torch.cuda.synchronize()
for b in range(1, B):
    buf[b * 3 * T:(b + 1) * 3 * T] = buf[:3 * T]
torch.cuda.synchronize()
for _ in range(3):
    run("SSSSM", [1, 0, 2])  # (A_ik factor, A_kj top, A_ij bot): see kernels.py access order
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run("SSSSM", [1, 0, 2])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"batch {B}: {ms:.3f} ms, {B * 2 * nb**3 / ms / 1e9:.1f} TF/s")
