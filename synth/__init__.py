"""Seeded synthetic inputs and weights for the GlassNet hot path (harness, not product).

This module is the ONE thing the oracle (``oracle/``) and the CUDA path
(``paper_2405_19056_b200``) share: it draws the input frames and the weight blob.
It holds none of the method's arithmetic (no normalisation, no layers, no pooling).

Recipe (stated in DESIGN.md §Inputs, following SURVEY.md §8(d) and BASELINE.json
configs[0]):

* Counter hash: ``h = splitmix64(splitmix64(seed*16 + stream) ^ counter)`` with
  ``counter = ((frame*H*W + y*W + x) << 10) | draw``.  Tile-invariant: a row band of a
  frame draws bitwise the same values as the full frame.  Stream ids: 1 gbuf, 2 direct,
  3 tbuf, 4 tcount, 5 c2 disc mask.
* ``u = (h >> 40) * 2^-24``; ``U[lo,hi] = lo + span*u`` in fp64.
* Gaussian ``z`` = Irwin-Hall sum of 12 uniforms (the four 16-bit fields of 3 hashes,
  each ``(f + 0.5)/65536``) minus 6 -- exact in fp64, no transcendental, so numpy and
  CUDA draw bitwise-identical values.
* Lognormal(mu=-1, sigma=1) = ``exp_ieee(-1 + z)`` where ``exp_ieee`` is a
  range-reduced degree-13 Taylor polynomial evaluated with separately rounded fp64
  ``*`` and ``+`` (no FMA) and ``ldexp`` -- again bitwise reproducible on both sides.
* Each value is rounded once fp64 -> fp32 (RNE), then fp32 -> bf16 (RNE) for bf16
  storage.
* Weights (host only): ``W ~ N(0, 2/fan_in)`` by Box-Muller in fp64, ``b ~ U(+-1/sqrt(fan_in))``;
  splitmix64 counter stream per (seed, layer index).

The device twin of the input generator lives in ``synth/synth_dev.cu``
(``libglassnet_synth.so``); ``tests/test_synth.py`` pins the two together bitwise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

STREAM_GBUF, STREAM_DIRECT, STREAM_TBUF, STREAM_TCOUNT, STREAM_DISC = 1, 2, 3, 4, 5

# Literal fp64 constants shared (by value) with synth_dev.cu.
POS_LO, POS_SPAN = -10.0, 20.0
DEPTH_LO, DEPTH_SPAN = 0.1, 99.9
ALPHA_LO, ALPHA_SPAN = 0.05, 0.9
LN_MU = -1.0
INV_LN2 = 1.4426950408889634
LN2_HI = 0.6931471803691238       # 0x3FE62E42FEE00000, trailing zeros -> k*LN2_HI exact
LN2_LO = 1.9082149292705877e-10   # 0x3DEA39EF35793C76
EXP_COEF = [1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664,
            0.008333333333333333, 0.001388888888888889, 0.0001984126984126984,
            2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07,
            2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10]

GBUF_CH, DIRECT_CH, REC_CH = 12, 3, 11
DRAWS_PER_SLOT = 32  # draw index j = slot*32 + d  (K <= 16 -> j < 512 < 1024)


# --------------------------------------------------------------------------- hashing
def splitmix64_int(x: int) -> int:
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> int:
    return splitmix64_int((seed * 16 + stream) & MASK64)


def _hash(key: int, base: np.ndarray, draw: int) -> np.ndarray:
    """base = (frame*H*W + pixel) << 10 (uint64 array)."""
    return splitmix64(np.uint64(key) ^ (base | np.uint64(draw)))


def u24(h: np.ndarray) -> np.ndarray:
    return (h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


def uniform(h, lo, span):
    return lo + span * u24(h)


def gauss(h0, h1, h2) -> np.ndarray:
    s = np.zeros(h0.shape, np.float64)
    for h in (h0, h1, h2):
        for sh in (0, 16, 32, 48):
            f = ((h >> np.uint64(sh)) & np.uint64(0xFFFF)).astype(np.float64)
            s = s + (f + 0.5) / 65536.0
    return s - 6.0


def exp_ieee(x: np.ndarray) -> np.ndarray:
    k = np.floor(x * INV_LN2 + 0.5)
    r = (x - k * LN2_HI) - k * LN2_LO
    p = np.full(x.shape, EXP_COEF[13])
    for j in range(12, -1, -1):
        p = p * r + EXP_COEF[j]
    return np.ldexp(p, k.astype(np.int32))


# --------------------------------------------------------------------------- rounding
def f64_to_f32(x: np.ndarray) -> np.ndarray:
    return x.astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """fp64/fp32 -> nearest bf16 value, returned as fp32 (via fp32, RNE both steps)."""
    return bf16_bits_to_f32(f32_to_bf16_bits(f64_to_f32(np.asarray(x, np.float64))))


# --------------------------------------------------------------------------- configs
@dataclass
class Config:
    name: str
    height: int
    width: int
    batch: int
    k_slots: int
    levels: int
    widths: tuple
    t_hidden: int
    precision: str           # "fp32" | "bf16"
    tcount_mode: str = "uniform"   # "uniform" n~U{0..K} | "discs" (c2)
    pool: str = "sum"
    notes: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c0": Config("c0", 64, 64, 1, 4, 3, (16, 32, 64), 32, "fp32",
                 notes="BASELINE.json configs[0]: tiny CPU-checkable frame, fp32 check mode"),
    "c1": Config("c1", 512, 512, 4, 8, 4, (32, 64, 128, 256), 64, "bf16",
                 notes="BASELINE.json configs[1]"),
    "c2": Config("c2", 720, 1280, 1, 8, 4, (32, 64, 128, 256), 64, "bf16", tcount_mode="discs",
                 notes="BASELINE.json configs[2]: 30% of pixels n=0 (union-of-discs mask)"),
    "c3": Config("c3", 1080, 1920, 32, 8, 4, (32, 64, 128, 256), 64, "bf16",
                 notes="BASELINE.json configs[3]: the metric's workload"),
    "c4": Config("c4", 2160, 3840, 1, 16, 4, (32, 64, 128, 256), 64, "bf16",
                 notes="BASELINE.json configs[4]: row-tile sharded frame"),
}


# --------------------------------------------------------------------------- weights
def layer_shapes(widths, levels, t_hidden, r_takes_ld=True, sigma_cond=False, pe_L=0, objects=False):
    """(name, W shape, fan_in) in blob order (SURVEY.md §8(b) 'Weights blob').  sigma_cond
    (SURVEY §8(f) N1): h's first layer also takes sigma = e0 at the pixel, T1.W [h][11 + c0].
    pe_L (N2): the inputs are positionally encoded, 11 -> 11(2L+1), 15 -> 15(2L+1) channels."""
    c = list(widths)[:levels]
    h = t_hidden
    pe = 2 * pe_L + 1
    n1 = 11 * pe + (c[0] if sigma_cond else 0)
    if objects:   # N4: h's layers are 3x3 convolutions (OHWI)
        out = [("T1", (h, 3, 3, 11), 99), ("T2", (h, 3, 3, h), 9 * h)]
    else:
        out = [("T1", (h, n1), n1), ("T2", (h, h), h)]
    cin = 15 * pe
    for lv in range(levels):
        out.append((f"F{lv}", (c[lv], 3, 3, cin), 9 * cin))
        cin = c[lv]
    out.append(("B", (c[0], c[0] + h + 1), c[0] + h + 1))
    for lv in range(levels - 1, 0, -1):
        out.append((f"R{lv}", (c[lv - 1], 3, 3, c[lv]), 9 * c[lv]))
    nin = c[0] + (3 if r_takes_ld else 0)
    out.append(("O", (3, nin), nin))
    return out


def weight_count(widths, levels, t_hidden, r_takes_ld=True, sigma_cond=False, pe_L=0, objects=False):
    n = 0
    for _, shp, _ in layer_shapes(widths, levels, t_hidden, r_takes_ld, sigma_cond, pe_L, objects):
        n += int(np.prod(shp)) + shp[0]
    return n


def make_weights(widths, levels, t_hidden, seed=0, r_takes_ld=True, bf16_weights=False, sigma_cond=False, pe_L=0,
                 objects=False):
    """Flat little-endian fp32 blob.  If bf16_weights, every W tensor (not the biases)
    is rounded RNE to a bf16-representable fp32 (SURVEY.md §8(c) preamble)."""
    parts = []
    for li, (_, shp, fan_in) in enumerate(layer_shapes(widths, levels, t_hidden, r_takes_ld, sigma_cond, pe_L, objects)):
        key = splitmix64_int((seed * 4096 + 1000 + li) & MASK64)
        nW = int(np.prod(shp))
        idx = np.arange(nW, dtype=np.uint64)
        h1 = splitmix64(np.uint64(key) ^ (idx * np.uint64(2)))
        h2 = splitmix64(np.uint64(key) ^ (idx * np.uint64(2) + np.uint64(1)))
        u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
        u2 = (h2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
        W = (z * math.sqrt(2.0 / fan_in)).astype(np.float32)
        if bf16_weights:
            W = round_to_bf16(W)
        nb = shp[0]
        hb = splitmix64(np.uint64(key) ^ (np.arange(nb, dtype=np.uint64) + np.uint64(1 << 40)))
        bound = 1.0 / math.sqrt(fan_in)
        b = (-bound + 2.0 * bound * u24(hb)).astype(np.float32)
        parts += [W.reshape(-1), b]
    return np.concatenate(parts).astype("<f4")


def ss_layer_shapes(s):
    """N3 super-sampler S (reading N3): (name, W shape, fan_in) in blob order."""
    return [("S1", (s, 3, 3, 15), 9 * 15), ("S2", (s, 3, 3, s), 9 * s), ("S3", (3, s), s)]


SS_RESIDUAL_SCALE = 0.1   # S3 (the residual head) drawn He-normal x 0.1: a near-identity init


def make_ss_weights(s, seed=0, bf16_weights=False):
    """Flat fp32 blob of S (S1.W S1.b S2.W S2.b S3.W S3.b); same generator as make_weights
    with layer keys 2000+li; the residual head scaled by SS_RESIDUAL_SCALE."""
    parts = []
    for li, (name, shp, fan_in) in enumerate(ss_layer_shapes(s)):
        key = splitmix64_int((seed * 4096 + 2000 + li) & MASK64)
        nW = int(np.prod(shp))
        idx = np.arange(nW, dtype=np.uint64)
        h1 = splitmix64(np.uint64(key) ^ (idx * np.uint64(2)))
        h2 = splitmix64(np.uint64(key) ^ (idx * np.uint64(2) + np.uint64(1)))
        u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
        u2 = (h2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
        sc = SS_RESIDUAL_SCALE if name == "S3" else 1.0
        W = (z * math.sqrt(2.0 / fan_in) * sc).astype(np.float32)
        if bf16_weights:
            W = round_to_bf16(W)
        hb = splitmix64(np.uint64(key) ^ (np.arange(shp[0], dtype=np.uint64) + np.uint64(1 << 40)))
        bound = sc / math.sqrt(fan_in)
        b = (-bound + 2.0 * bound * u24(hb)).astype(np.float32)
        parts += [W.reshape(-1), b]
    return np.concatenate(parts).astype("<f4")


def gen_image(seed, nframes, H, W):
    """A [0,1] RGB image batch standing in for GlassNet's output (S's input in isolation)."""
    key = stream_key(seed, 6)
    b = _bases(0, nframes, H, W, 0, H, 0, W)
    return np.stack([u24(_hash(key, b, c)) for c in range(3)], axis=-1).astype(np.float32)


def gen_gbuf_hi(seed, nframes, H2, W2, precision):
    """The hi-res G-buffer S reads: the G-buffer recipe on the 2H x 2W grid (seed distinct from
    the low-res frame's), stored in `precision`."""
    return store(gen_gbuf64(seed, 0, nframes, H2, W2, 0, H2, 0, W2), precision)


# --------------------------------------------------------------------------- inputs
def _bases(frame0, nframes, H, W, y0, y1, x0, x1):
    f = np.arange(frame0, frame0 + nframes, dtype=np.uint64)[:, None, None]
    y = np.arange(y0, y1, dtype=np.uint64)[None, :, None]
    x = np.arange(x0, x1, dtype=np.uint64)[None, None, :]
    pix = f * np.uint64(H * W) + y * np.uint64(W) + x
    return pix << np.uint64(10)


def _normal3(key, base, d0):
    z = [gauss(_hash(key, base, d0 + 3 * c), _hash(key, base, d0 + 3 * c + 1),
               _hash(key, base, d0 + 3 * c + 2)) for c in range(3)]
    n2 = (z[0] * z[0] + z[1] * z[1]) + z[2] * z[2]
    nrm = np.sqrt(n2)
    small = nrm < 1e-12
    safe = np.where(small, 1.0, nrm)
    out = [np.where(small, 0.0, z[0] / safe), np.where(small, 0.0, z[1] / safe),
           np.where(small, 1.0, z[2] / safe)]
    return out


def _lognormal(key, base, d0):
    z = gauss(_hash(key, base, d0), _hash(key, base, d0 + 1), _hash(key, base, d0 + 2))
    return exp_ieee(LN_MU + z)


def gen_gbuf64(seed, frame0, nframes, H, W, y0, y1, x0, x1):
    key = stream_key(seed, STREAM_GBUF)
    b = _bases(frame0, nframes, H, W, y0, y1, x0, x1)
    ch = [uniform(_hash(key, b, d), POS_LO, POS_SPAN) for d in range(3)]
    ch += _normal3(key, b, 3)                                         # draws 3..11
    ch += [u24(_hash(key, b, 12 + d)) for d in range(3)]              # albedo
    ch += [u24(_hash(key, b, 15)), u24(_hash(key, b, 16))]            # roughness, metallic
    ch += [uniform(_hash(key, b, 17), DEPTH_LO, DEPTH_SPAN)]          # depth
    return np.stack(ch, axis=-1)


def gen_direct64(seed, frame0, nframes, H, W, y0, y1, x0, x1):
    key = stream_key(seed, STREAM_DIRECT)
    b = _bases(frame0, nframes, H, W, y0, y1, x0, x1)
    return np.stack([_lognormal(key, b, 3 * c) for c in range(3)], axis=-1)


def gen_tbuf64(seed, frame0, nframes, H, W, K, y0, y1, x0, x1):
    key = stream_key(seed, STREAM_TBUF)
    b = _bases(frame0, nframes, H, W, y0, y1, x0, x1)
    slots = []
    for k in range(K):
        d = k * DRAWS_PER_SLOT
        ch = _normal3(key, b, d)                                      # d+0..8
        ch += [u24(_hash(key, b, d + 9 + c)) for c in range(3)]       # colour
        ch += [uniform(_hash(key, b, d + 12), ALPHA_LO, ALPHA_SPAN)]  # alpha
        ch += [uniform(_hash(key, b, d + 13), DEPTH_LO, DEPTH_SPAN)]  # depth
        ch += [_lognormal(key, b, d + 14 + 3 * c) for c in range(3)]  # direct d+14..22
        slots.append(np.stack(ch, axis=-1))
    return np.stack(slots, axis=-2)


def disc_mask(seed, H, W, K=None, coverage=0.7, max_discs=4096):
    """c2's spatial mask: union of random discs (centres uniform, radii U[H/16, H/4]) added
    until >= coverage of the pixels are covered."""
    key = stream_key(seed, STREAM_DISC)
    yy, xx = np.mgrid[0:H, 0:W]
    cov = np.zeros((H, W), bool)
    for i in range(max_discs):
        hs = [splitmix64(np.array([key ^ ((i << 2) | d)], np.uint64))[0] for d in range(3)]
        cx = float((int(hs[0]) >> 40) * 2.0 ** -24) * W
        cy = float((int(hs[1]) >> 40) * 2.0 ** -24) * H
        r = H / 16.0 + (H / 4.0 - H / 16.0) * float((int(hs[2]) >> 40) * 2.0 ** -24)
        cov |= (xx + 0.5 - cx) ** 2 + (yy + 0.5 - cy) ** 2 <= r * r
        if cov.mean() >= coverage:
            break
    return cov


def gen_tcount(seed, frame0, nframes, H, W, K, y0, y1, x0, x1, mask=None):
    """n ~ U{0..K} (integer, exact); with a mask: covered -> U{1..K}, else 0."""
    key = stream_key(seed, STREAM_TCOUNT)
    b = _bases(frame0, nframes, H, W, y0, y1, x0, x1)
    t = _hash(key, b, 0) >> np.uint64(40)
    if mask is None:
        n = (t * np.uint64(K + 1)) >> np.uint64(24)
    else:
        n = np.uint64(1) + ((t * np.uint64(K)) >> np.uint64(24))
        n = np.where(mask[None, y0:y1, x0:x1], n, np.uint64(0))
    return n.astype(np.uint8)


@dataclass
class Frames:
    """Inputs as stored (fp32 arrays or bf16 bit patterns as uint16) plus fp64 views."""
    gbuf: np.ndarray
    direct: np.ndarray
    tbuf: np.ndarray
    tcount: np.ndarray
    precision: str

    def as64(self):
        f = (lambda a: bf16_bits_to_f32(a).astype(np.float64)) if self.precision == "bf16" \
            else (lambda a: a.astype(np.float64))
        return f(self.gbuf), f(self.direct), f(self.tbuf), self.tcount


def store(x64: np.ndarray, precision: str) -> np.ndarray:
    x32 = f64_to_f32(x64)
    return f32_to_bf16_bits(x32) if precision == "bf16" else x32


def gen_frames(cfg: Config, seed=1, frame0=0, nframes=None, rows=None, cols=None, mask=None):
    """Generate frames [frame0, frame0+nframes) restricted to rows/cols windows (global
    coordinates; tile-invariant)."""
    H, W, K = cfg.height, cfg.width, cfg.k_slots
    nframes = cfg.batch if nframes is None else nframes
    y0, y1 = rows if rows is not None else (0, H)
    x0, x1 = cols if cols is not None else (0, W)
    if cfg.tcount_mode == "discs" and mask is None:
        mask = disc_mask(seed, H, W)
    g = store(gen_gbuf64(seed, frame0, nframes, H, W, y0, y1, x0, x1), cfg.precision)
    d = store(gen_direct64(seed, frame0, nframes, H, W, y0, y1, x0, x1), cfg.precision)
    t = store(gen_tbuf64(seed, frame0, nframes, H, W, K, y0, y1, x0, x1), cfg.precision)
    n = gen_tcount(seed, frame0, nframes, H, W, K, y0, y1, x0, x1,
                   mask if cfg.tcount_mode == "discs" else None)
    return Frames(g, d, t, n, cfg.precision)
