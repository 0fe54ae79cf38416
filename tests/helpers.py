"""Test helpers: host<->torch marshalling and the windowed oracle for sampled full-size parity."""
import numpy as np

import oracle
import synth

BF16_TOL = (3e-2, 3e-3)    # BASELINE.json north_star: max abs, mean abs on the [0,1] output (bf16 mode)
FP32_TOL = 1e-4            # fp32 check mode


def to_torch(fr, device="cuda"):
    import torch
    if fr.precision == "bf16":
        cv = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)
    else:
        cv = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    g, d, t = (cv(a).to(device) for a in (fr.gbuf, fr.direct, fr.tbuf))
    n = torch.from_numpy(np.ascontiguousarray(fr.tcount)).to(device)
    return g, d, t, n


def sigma_of(cfg):
    return bool(cfg.extra.get("sigma_cond", False))


def pe_of(cfg):
    return int(cfg.extra.get("pe_L", 0))


def weights_for(cfg, seed=0):
    return synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=seed,
                              bf16_weights=(cfg.precision == "bf16"), sigma_cond=sigma_of(cfg), pe_L=pe_of(cfg))


def net_for(cfg, max_batch=None, **kw):
    from paper_2405_19056_b200 import GlassNet, make_dims
    dims = make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels,
                     precision=cfg.precision, max_batch=cfg.batch if max_batch is None else max_batch,
                     pool=cfg.pool, sigma_cond=sigma_of(cfg), pe_L=pe_of(cfg), **kw)
    return GlassNet(weights_for(cfg), dims)


def oracle_full(cfg, weights, fr, frame_idx=0):
    g, d, t, n = fr.as64()
    dims = oracle.dims_from_cfg(cfg)
    return oracle.forward(dims, weights.astype(np.float64), g[frame_idx], d[frame_idx], t[frame_idx],
                          n[frame_idx])


def window_oracle(cfg, weights, frame, rows, cols, margin=64, seed=1, mask=None):
    """Oracle output for out[frame, rows[0]:rows[1], cols[0]:cols[1]] computed on a crop of
    the frame extended by `margin` px (aligned to 2^(L-1)); inputs drawn by the host
    generator for exactly that crop (tile-invariant).  Bitwise equal to the full-frame
    oracle when margin covers the receptive field (pinned in test_window_oracle)."""
    u = 1 << (cfg.levels - 1)
    H, W = cfg.height, cfg.width
    a = max(0, (rows[0] - margin) // u * u)
    b = min(H, -(-(rows[1] + margin) // u) * u)
    c = max(0, (cols[0] - margin) // u * u)
    e = min(W, -(-(cols[1] + margin) // u) * u)
    fr = synth.gen_frames(cfg, seed=seed, frame0=frame, nframes=1, rows=(a, b), cols=(c, e), mask=mask)
    g, d, t, n = fr.as64()
    dims = oracle.make_dims(b - a, e - c, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, pool=cfg.pool,
                            sigma_cond=sigma_of(cfg), pe_L=pe_of(cfg))
    out = oracle.forward(dims, weights.astype(np.float64), g[0], d[0], t[0], n[0])
    return out[rows[0] - a:rows[1] - a, cols[0] - c:cols[1] - c]


def errs(gpu, ref):
    e = np.abs(np.asarray(gpu, np.float64) - ref)
    return float(e.max()), float(e.mean())


def _crop(H, W, u, rows, cols, margin):
    a = max(0, (rows[0] - margin) // u * u)
    b = min(H, -(-(rows[1] + margin) // u) * u)
    c = max(0, (cols[0] - margin) // u * u)
    e = min(W, -(-(cols[1] + margin) // u) * u)
    return a, b, c, e


def band_oracle(cfg, weights, fr, frame_idx=0, margin=40, threads=None, band=None):
    """Full-frame oracle output of frame `frame_idx` of the stored inputs `fr` (synth.Frames),
    computed as row bands of the frame, each from a crop extended by `margin` rows (aligned to
    2^(L-1)), in a thread pool (the C oracle releases the GIL).  Bitwise equal to the
    full-frame oracle when the margin covers the receptive field (pinned in
    test_window_oracle.py for margin 40)."""
    import concurrent.futures as cf
    import os
    H, W, L = cfg.height, cfg.width, cfg.levels
    u = 1 << (L - 1)
    threads = threads or max(1, os.cpu_count() or 1)
    if band is None:
        band = max(u, -(-H // (2 * threads)) // u * u)
    w64 = weights.astype(np.float64)
    out = np.zeros((H, W, 3), np.float64)

    def run(r0):
        r1 = min(H, r0 + band)
        a, b, _, _ = _crop(H, W, u, (r0, r1), (0, W), margin)
        sub = synth.Frames(fr.gbuf[frame_idx:frame_idx + 1, a:b], fr.direct[frame_idx:frame_idx + 1, a:b],
                           fr.tbuf[frame_idx:frame_idx + 1, a:b], fr.tcount[frame_idx:frame_idx + 1, a:b],
                           fr.precision)
        g, d, t, n = sub.as64()
        dims = oracle.make_dims(b - a, W, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, pool=cfg.pool,
                                sigma_cond=sigma_of(cfg), pe_L=pe_of(cfg))
        o = oracle.forward(dims, w64, g[0], d[0], t[0], n[0])
        out[r0:r1] = o[r0 - a:r1 - a]

    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(0, H, band)))
    return out


def frames_from_device(g, d, t, n, precision="bf16"):
    """Device input tensors -> synth.Frames of their stored bits (host)."""
    import torch
    if precision == "bf16":
        cv = lambda x: x.cpu().view(torch.int16).numpy().view(np.uint16)
    else:
        cv = lambda x: x.cpu().numpy()
    return synth.Frames(cv(g), cv(d), cv(t), n.cpu().numpy(), precision)


def ss_band_oracle(s, w_ss, img, gbuf_hi, band=None, threads=None, input_norm=True):
    """Oracle S (N3) of one frame as low-res row bands, each from a crop extended by one low-res
    row (= two hi-res rows, the receptive field of S's two 3x3 convs) in a thread pool.  Bitwise
    equal to the whole-frame oracle (pinned in test_oracle_ss_pins.py)."""
    import concurrent.futures as cf
    import os
    import oracle
    H, W, _ = img.shape
    threads = threads or max(1, os.cpu_count() or 1)
    band = band or max(1, -(-H // (2 * threads)))
    out = np.zeros((2 * H, 2 * W, 3), np.float64)

    def run(r0):
        r1 = min(H, r0 + band)
        a, b = max(0, r0 - 1), min(H, r1 + 1)
        o = oracle.supersample(s, w_ss, img[a:b], gbuf_hi[2 * a:2 * b], input_norm=input_norm)
        out[2 * r0:2 * r1] = o[2 * (r0 - a):2 * (r1 - a)]

    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(0, H, band)))
    return out
