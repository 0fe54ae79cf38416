"""ctypes wrapper of the fp64 CPU oracle (oracle/glassnet_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product package
(paper_2405_19056_b200) never imports it and shares no code with it.

Parity status per function:
  og_conv3x3  pinned (P2 Toeplitz, P7 identity, P8 stride, torch conv2d)
  og_up2      pinned (P9 constant / ramp closed form / torch interpolate)
  og_T_pixel  pinned (P1 hand-expanded golden, P3 permutation, P4 garbage, P5 empty, P6 duplicate);
              sigma_cond (N1) pinned by P1s (hand-expanded golden with sigma), P15 (zero sigma
              weights = the unconditioned network, bitwise) and P16 (records with zero weights:
              every fragment is h(sigma), n = 2 gives exactly 2 h(sigma)) and P10 (torch-fp64)
  og_forward  pinned (P10 torch-fp64 composition, P11 homogeneity, P13 tiles, P14 shift)
  og_posenc (N2) pinned (PE1 SPEC S:401-403 examples, PE2 channel count, PE3 torch sin/cos at
              exact dyadic points); forward with pe_L pinned by P15pe (zero sin/cos weights = the
              unencoded network, bitwise) and P10pe (torch-fp64 composition with torch.sin/cos PE)
  og_forward_objects (N4) pinned (P17 centre-tap convs = the pixel-major network on the slot
              decomposition, bitwise; PO1 object order bitwise; PO2 garbage outside the coverage
              bitwise; PO3 locality of an object's contribution; PO4 tau == torch-fp64 conv2d sum)
  og_supersample (N3) pinned (PS1 identity residual = nearest up-sampling, PS2 constant residual
              = clamp(u + beta), PS3 torch-fp64 composition (interpolate nearest + conv2d),
              PS4 receptive field: a coarse pixel reaches only hi-res pixels within 2 of its block)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "glassnet_oracle.c")
_LIB = os.path.join(_HERE, "libglassnet_oracle.so")
_lib = None


def build(force=False):
    """gcc -O2, no fast-math, no FP contraction."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Dims(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int), ("W", ctypes.c_int), ("K", ctypes.c_int), ("L", ctypes.c_int),
                ("c", ctypes.c_int * 4), ("h", ctypes.c_int), ("pool", ctypes.c_int),
                ("r_takes_ld", ctypes.c_int), ("input_norm", ctypes.c_int), ("sigma_cond", ctypes.c_int),
                ("pe_L", ctypes.c_int), ("objects", ctypes.c_int)]


_P = ctypes.POINTER(ctypes.c_double)


class Dump(ctypes.Structure):
    _fields_ = [("x", _P), ("e", _P * 4), ("tau", _P), ("phi", _P), ("y", _P * 4),
                ("d", _P * 4), ("logits", _P)]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _lib.og_weight_count.restype = ctypes.c_size_t
        _lib.og_weight_count.argtypes = [ctypes.POINTER(Dims)]
        _lib.og_forward.restype = ctypes.c_int
        _lib.og_conv3x3.restype = None
        _lib.og_up2.restype = None
        _lib.og_T_pixel.restype = None
        _lib.og_posenc.restype = None
        _lib.og_ss_weight_count.restype = ctypes.c_size_t
        _lib.og_ss_weight_count.argtypes = [ctypes.c_int]
        _lib.og_supersample.restype = ctypes.c_int
    return _lib


def make_dims(H, W, K, widths, t_hidden, levels=None, pool="sum", r_takes_ld=True,
              input_norm=True, sigma_cond=False, pe_L=0, objects=False) -> Dims:
    levels = len(widths) if levels is None else levels
    c = (ctypes.c_int * 4)(*(list(widths) + [0] * (4 - len(widths))))
    return Dims(H, W, K, levels, c, t_hidden, 1 if pool == "mean" else 0,
                1 if r_takes_ld else 0, 1 if input_norm else 0, 1 if sigma_cond else 0, int(pe_L),
                1 if objects else 0)


def dims_from_cfg(cfg, H=None, W=None, **kw) -> Dims:
    kw.setdefault("sigma_cond", bool(getattr(cfg, "extra", {}).get("sigma_cond", False)))
    kw.setdefault("pe_L", int(getattr(cfg, "extra", {}).get("pe_L", 0)))
    kw.setdefault("objects", bool(getattr(cfg, "extra", {}).get("objects", False)))
    return make_dims(cfg.height if H is None else H, cfg.width if W is None else W,
                     cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, pool=cfg.pool, **kw)


def _ptr(a):
    return a.ctypes.data_as(_P)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def weight_count(d: Dims) -> int:
    return int(lib().og_weight_count(ctypes.byref(d)))


def lvl(n, l):
    for _ in range(l):
        n = (n + 1) // 2
    return n


def forward(d: Dims, weights, gbuf, direct, tbuf, tcount, dump=False):
    """One frame (arrays without batch dim), or a batch (leading dim) -> out fp64."""
    gbuf = np.asarray(gbuf)
    if gbuf.ndim == 4:
        res = [forward(d, weights, gbuf[b], direct[b], tbuf[b], tcount[b], dump)
               for b in range(gbuf.shape[0])]
        if dump:
            return np.stack([r[0] for r in res]), [r[1] for r in res]
        return np.stack(res)
    H, W, L, h = d.H, d.W, d.L, d.h
    w = _c64(weights)
    assert w.size == weight_count(d), (w.size, weight_count(d))
    g, dr, t = _c64(gbuf), _c64(direct), _c64(tbuf)
    n = np.ascontiguousarray(tcount, dtype=np.uint8)
    assert g.shape == (H, W, 12) and dr.shape == (H, W, 3) and t.shape == (H, W, d.K, 11)
    out = np.zeros((H, W, 3), np.float64)
    dm = None
    arrays = {}
    if dump:
        c = list(d.c)
        arrays["x"] = np.zeros((H, W, 15 * (2 * d.pe_L + 1)))
        arrays["e"] = [np.zeros((lvl(H, l), lvl(W, l), c[l])) for l in range(L)]
        arrays["tau"] = np.zeros((H, W, h + 1))
        arrays["phi"] = np.zeros((H, W, c[0]))
        arrays["y"] = [None] + [np.zeros((lvl(H, l), lvl(W, l), c[l - 1])) for l in range(1, L)]
        arrays["d"] = [np.zeros((lvl(H, l), lvl(W, l), c[l])) for l in range(L - 1)]
        arrays["logits"] = np.zeros((H, W, 3))
        dm = Dump()
        dm.x, dm.tau, dm.phi, dm.logits = (_ptr(arrays[k]) for k in ("x", "tau", "phi", "logits"))
        for l in range(L):
            dm.e[l] = _ptr(arrays["e"][l])
        for l in range(1, L):
            dm.y[l] = _ptr(arrays["y"][l])
        for l in range(L - 1):
            dm.d[l] = _ptr(arrays["d"][l])
    rc = lib().og_forward(ctypes.byref(d), _ptr(w), _ptr(g), _ptr(dr), _ptr(t),
                          n.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), _ptr(out),
                          ctypes.byref(dm) if dm is not None else None)
    if rc != 0:
        raise RuntimeError(f"og_forward failed rc={rc}")
    return (out, arrays) if dump else out


def conv3x3(x, Wt, b, stride=1, relu=True):
    x, Wt, b = _c64(x), _c64(Wt), _c64(b)
    H, W, Cin = x.shape
    Cout = Wt.shape[0]
    assert Wt.shape == (Cout, 3, 3, Cin)
    out = np.zeros(((H + stride - 1) // stride, (W + stride - 1) // stride, Cout))
    lib().og_conv3x3(_ptr(x), H, W, Cin, _ptr(Wt), _ptr(b), Cout, stride, int(relu), _ptr(out))
    return out


def up2(v, H2, W2):
    v = _c64(v)
    h, w, C = v.shape
    out = np.zeros((H2, W2, C))
    lib().og_up2(_ptr(v), h, w, C, H2, W2, _ptr(out))
    return out


def T_pixel(d: Dims, W1, b1, W2, b2, records, n, sigma=None):
    """tau of one pixel; sigma [c0] = the scene features (used only when d.sigma_cond)."""
    rec = _c64(records)
    assert rec.shape == (d.K, 11)
    W1, b1, W2, b2 = _c64(W1), _c64(b1), _c64(W2), _c64(b2)
    sg = _c64(np.zeros(max(d.c[0], 1)) if sigma is None else sigma)
    if d.sigma_cond:
        assert sigma is not None and sg.shape == (d.c[0],)
    tau = np.zeros(d.h + 1)
    lib().og_T_pixel(ctypes.byref(d), _ptr(W1), _ptr(b1), _ptr(W2), _ptr(b2), _ptr(rec),
                     int(n), _ptr(sg), _ptr(tau))
    return tau


def split_weights(d: Dims, weights):
    """Blob -> dict of fp64 arrays (same documented order the library parses)."""
    w = _c64(weights)
    h, L, c = d.h, d.L, list(d.c)
    out, p = {}, 0

    def take(name, shape):
        nonlocal p
        n = int(np.prod(shape))
        out[name] = w[p:p + n].reshape(shape)
        p += n

    pe = 2 * d.pe_L + 1
    if d.objects:   # N4: h's layers are 3x3 convolutions (OHWI)
        take("T1.W", (h, 3, 3, 11)); take("T1.b", (h,)); take("T2.W", (h, 3, 3, h)); take("T2.b", (h,))
    else:
        take("T1.W", (h, 11 * pe + (c[0] if d.sigma_cond else 0))); take("T1.b", (h,)); take("T2.W", (h, h))
        take("T2.b", (h,))
    cin = 15 * pe
    for l in range(L):
        take(f"F{l}.W", (c[l], 3, 3, cin)); take(f"F{l}.b", (c[l],)); cin = c[l]
    take("B.W", (c[0], c[0] + h + 1)); take("B.b", (c[0],))
    for l in range(L - 1, 0, -1):
        take(f"R{l}.W", (c[l - 1], 3, 3, c[l])); take(f"R{l}.b", (c[l - 1],))
    nO = c[0] + (3 if d.r_takes_ld else 0)
    take("O.W", (3, nO)); take("O.b", (3,))
    assert p == w.size
    return out


def ss_weight_count(s: int) -> int:
    return int(lib().og_ss_weight_count(int(s)))


def supersample(s, weights_ss, img, gbuf_hi, input_norm=True):
    """N3 super-sampler S of one frame (or a batch): img [H][W][3], gbuf_hi [2H][2W][12] ->
    out [2H][2W][3] fp64 (glassnet_oracle.c og_supersample; reading N3)."""
    img = np.asarray(img)
    if img.ndim == 4:
        return np.stack([supersample(s, weights_ss, img[b], gbuf_hi[b], input_norm) for b in range(img.shape[0])])
    H, W, _ = img.shape
    w, im, g = _c64(weights_ss), _c64(img), _c64(gbuf_hi)
    assert w.size == ss_weight_count(s), (w.size, ss_weight_count(s))
    assert im.shape == (H, W, 3) and g.shape == (2 * H, 2 * W, 12)
    out = np.zeros((2 * H, 2 * W, 3))
    rc = lib().og_supersample(H, W, int(s), int(bool(input_norm)), _ptr(w), _ptr(im), _ptr(g), _ptr(out))
    if rc != 0:
        raise RuntimeError(f"og_supersample failed rc={rc}")
    return out


def split_ss_weights(s, weights_ss):
    w = _c64(weights_ss)
    out, p = {}, 0
    for name, shape in (("S1.W", (s, 3, 3, 15)), ("S1.b", (s,)), ("S2.W", (s, 3, 3, s)), ("S2.b", (s,)),
                        ("S3.W", (3, s)), ("S3.b", (3,))):
        n = int(np.prod(shape))
        out[name] = w[p:p + n].reshape(shape)
        p += n
    assert p == w.size
    return out


def posenc(v, L):
    """N2 gamma(v) per channel (og_posenc): [n] -> [n (2L + 1)] fp64."""
    v = _c64(np.atleast_1d(v))
    out = np.zeros(v.size * (2 * L + 1))
    lib().og_posenc(_ptr(v), int(v.size), int(L), _ptr(out))
    return out


def objects_from_slots(tbuf, tcount, K):
    """N4's synthetic object buffers: object k holds slot k of every pixel, covered where k < n
    (the pixel-major frame's information, object-major).  tbuf [H][W][K][11], tcount [H][W]."""
    objs = [np.ascontiguousarray(tbuf[:, :, k, :]) for k in range(K)]
    covs = [np.ascontiguousarray((np.asarray(tcount).astype(np.int64) > k).astype(np.uint8)) for k in range(K)]
    return objs, covs


def forward_objects(d: Dims, weights, gbuf, direct, objs, covers, dump=False):
    """N4: one frame from t object buffers objs[i] [H][W][11] and coverage covers[i] [H][W]."""
    H, W = d.H, d.W
    w = _c64(weights)
    assert d.objects and w.size == weight_count(d), (w.size, weight_count(d))
    g, dr = _c64(gbuf), _c64(direct)
    ob = [_c64(o) for o in objs]
    cv = [np.ascontiguousarray(c, dtype=np.uint8) for c in covers]
    t = len(ob)
    for o, c in zip(ob, cv):
        assert o.shape == (H, W, 11) and c.shape == (H, W)
    optr = (_P * max(t, 1))(*[_ptr(o) for o in ob])
    u8p = ctypes.POINTER(ctypes.c_uint8)
    cptr = (u8p * max(t, 1))(*[c.ctypes.data_as(u8p) for c in cv])
    out = np.zeros((H, W, 3))
    arrays, dm = {}, None
    if dump:
        arrays["tau"] = np.zeros((H, W, d.h + 1))
        dm = Dump()
        dm.tau = _ptr(arrays["tau"])
    rc = lib().og_forward_objects(ctypes.byref(d), _ptr(w), _ptr(g), _ptr(dr), t, optr, cptr, _ptr(out),
                                  ctypes.byref(dm) if dm is not None else None)
    if rc != 0:
        raise RuntimeError(f"og_forward_objects failed rc={rc}")
    return (out, arrays) if dump else out
