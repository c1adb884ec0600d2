"""Device-memory helpers for the GPU tests (torch is plumbing only)."""
import ctypes as C

import numpy as np
import torch

from paper_1402_6601_b200 import _native


def dev_tile(a: np.ndarray, extra: int = 0) -> torch.Tensor:
    """Column-major tile (+ optional side area) as a flat cuda float64 tensor."""
    flat = np.asfortranarray(a).ravel(order="F")
    t = torch.zeros(flat.size + extra, dtype=torch.float64, device="cuda")
    t[: flat.size] = torch.from_numpy(flat).cuda()
    return t


def host_tile(t: torch.Tensor, b: int) -> np.ndarray:
    return t[: b * b].cpu().numpy().reshape(b, b, order="F")


def tile_run(kind: int, tensors, nb: int, ib: int = 0) -> int:
    """Run one tile kernel through the C-ABI on torch's current stream; returns the status word."""
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ptrs = (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = _native.lib().hg_tile_run(kind, torch.cuda.current_device(), stream, ptrs, len(tensors), nb, ib,
                                   C.c_void_p(status.data_ptr()))
    _native.check(rc, "hg_tile_run")
    torch.cuda.synchronize()
    return int(status.item())
