"""Launch each tile kind a few times (for ncu): python tools/profile_kinds.py KIND [KIND ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import paper_1402_6601_b200 as H
from paper_1402_6601_b200 import _native

nb, ib = 1024, 128
kinds = sys.argv[1:] or ["POTRF", "TRSM"]
nts = {"POTRF": 1, "TRSM": 2, "SYRK": 2, "GEMM": 3, "GETRF_INC": 1, "GESSM": 2, "TSTRF": 2, "SSSSM": 3,
       "GEQRT": 1, "UNMQR": 2, "TSQRT": 2, "TSMQR": 3}
rng = np.random.default_rng(0)
status = torch.zeros(1, dtype=torch.int32, device="cuda")
for kind in kinds:
    n = nts[kind]
    ts = []
    for i in range(n):
        a = rng.uniform(-0.5, 0.5, (nb, nb))
        if i == 0:
            a = (a + a.T) / 2 + nb * np.eye(nb)
        t = torch.zeros(nb * nb + ib * nb + nb, dtype=torch.float64, device="cuda")
        t[: nb * nb] = torch.from_numpy(np.asfortranarray(a).ravel(order="F")).cuda()
        ts.append(t)
    ptrs = (C.c_void_p * n)(*[t.data_ptr() for t in ts])
    for _ in range(2):
        _native.check(_native.lib().hg_tile_run(H.ALL_KINDS.index(kind), 0, None, ptrs, n, nb, ib,
                                                C.c_void_p(status.data_ptr())), kind)
    torch.cuda.synchronize()
print("done")
