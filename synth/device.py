"""ctypes binding of synth/libglassnet_synth.so (device twin of the numpy generator)."""
from __future__ import annotations

import ctypes
import os

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libglassnet_synth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: build with __graft_entry__.build()")
        L = ctypes.CDLL(_LIB)
        L.glassnet_synth_fill.restype = ctypes.c_int
        L.glassnet_synth_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]
        _lib = L
    return _lib


def fill(cfg, gbuf, direct, tbuf, tcount, seed=1, frame0=0, rows=None, mask=None, stream=None):
    """Fill device tensors [nframes][rows][W][...] with frames frame0.. of cfg."""
    import torch
    nframes = gbuf.shape[0]
    y0, y1 = rows if rows is not None else (0, cfg.height)
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream.cuda_stream
    rc = lib().glassnet_synth_fill(0 if cfg.precision == "bf16" else 1, seed, frame0, nframes, cfg.height,
                                   cfg.width, cfg.k_slots, y0, y1, gbuf.data_ptr(), direct.data_ptr(),
                                   tbuf.data_ptr(), tcount.data_ptr(), 0 if mask is None else mask.data_ptr(), st)
    if rc != 0:
        raise RuntimeError(f"glassnet_synth_fill failed: cuda error {rc}")


def alloc_and_fill(cfg, nframes=None, seed=1, frame0=0, rows=None, mask=None, device="cuda"):
    import torch
    nframes = cfg.batch if nframes is None else nframes
    y0, y1 = rows if rows is not None else (0, cfg.height)
    Hr, W, K = y1 - y0, cfg.width, cfg.k_slots
    dt = torch.bfloat16 if cfg.precision == "bf16" else torch.float32
    g = torch.empty((nframes, Hr, W, 12), dtype=dt, device=device)
    d = torch.empty((nframes, Hr, W, 3), dtype=dt, device=device)
    t = torch.empty((nframes, Hr, W, K, 11), dtype=dt, device=device)
    n = torch.empty((nframes, Hr, W), dtype=torch.uint8, device=device)
    m = None
    if cfg.tcount_mode == "discs":
        import numpy as np
        import synth
        mm = synth.disc_mask(seed, cfg.height, cfg.width) if mask is None else mask
        m = torch.from_numpy(np.ascontiguousarray(mm).astype(np.uint8)).to(device)
    fill(cfg, g, d, t, n, seed=seed, frame0=frame0, rows=rows, mask=m)
    return g, d, t, n
