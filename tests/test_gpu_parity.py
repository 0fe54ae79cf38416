"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star): bf16 mode max abs <= 3e-2 and mean abs <= 3e-3 on
the [0,1] output; fp32 check mode max abs <= 1e-4.  Bitwise: slot permutation, masked
garbage, run-to-run determinism, kernel-family independence of the permutation property.
"""
import numpy as np
import pytest

import synth
from helpers import BF16_TOL, FP32_TOL, band_oracle, errs, frames_from_device, net_for, oracle_full, to_torch, weights_for

pytestmark = pytest.mark.gpu

C1NET = dict(levels=4, widths=(32, 64, 128, 256), t_hidden=64)
FAMILIES = ["tc", "simt"]


def _cfg(name, H, W, B, K, prec, net=None, **kw):
    n = net or C1NET
    return synth.Config(name, H, W, B, K, n["levels"], n["widths"], n["t_hidden"], prec, **kw)



def _run(cfg, fr, family=None, net=None):
    import torch
    net = net or net_for(cfg)
    if family is not None:
        net.set_kernel_family(family == "tc")
    g, d, t, n = to_torch(fr)
    out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    return out.cpu().numpy(), net


def test_synth_device_matches_numpy(cuda_ok):
    from synth import device
    for prec in ("bf16", "fp32"):
        cfg = _cfg("s", 40, 56, 2, 5, prec)
        host = synth.gen_frames(cfg, seed=7)
        g, d, t, n = device.alloc_and_fill(cfg, seed=7)
        dev = [a.cpu().view(__import__("torch").int16).numpy().view(np.uint16) if prec == "bf16" else a.cpu().numpy()
               for a in (g, d, t)]
        assert np.array_equal(dev[0], host.gbuf) and np.array_equal(dev[1], host.direct)
        assert np.array_equal(dev[2], host.tbuf) and np.array_equal(n.cpu().numpy(), host.tcount)
        # row window + frame offset
        g2, d2, t2, n2 = device.alloc_and_fill(cfg, nframes=1, seed=7, frame0=1, rows=(8, 24))
        assert np.array_equal(n2.cpu().numpy()[0], host.tcount[1, 8:24])
    # disc mask mode
    cfg = _cfg("s2", 48, 80, 1, 8, "bf16", tcount_mode="discs")
    m = synth.disc_mask(1, 48, 80)
    _, _, _, n = device.alloc_and_fill(cfg, mask=m)
    assert np.array_equal(n.cpu().numpy(), synth.gen_frames(cfg, mask=m).tcount)


def test_fp32_check_mode_c0(cuda_ok):
    """configs[0] (64x64, K=4, fp32): max abs <= 1e-4 (P15)."""
    cfg = synth.CONFIGS["c0"]
    fr = synth.gen_frames(cfg)
    out, _ = _run(cfg, fr)
    mx, mean = errs(out[0], oracle_full(cfg, weights_for(cfg), fr))
    print(f"c0 fp32: max {mx:.3e} mean {mean:.3e}")
    assert mx <= FP32_TOL


def test_fp32_check_mode_c1_net_ragged(cuda_ok):
    cfg = _cfg("f32", 40, 136, 2, 8, "fp32")
    fr = synth.gen_frames(cfg)
    out, _ = _run(cfg, fr)
    w = weights_for(cfg)
    for b in range(2):
        mx, _ = errs(out[b], oracle_full(cfg, w, fr, b))
        assert mx <= FP32_TOL, (b, mx)


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("H,W,K,B", [(64, 96, 8, 2), (40, 280, 8, 1), (32, 136, 16, 1), (24, 48, 3, 3)])
def test_bf16_parity_small(cuda_ok, family, H, W, K, B):
    """Several tiles plus ragged tails; c1 network; K in {3, 8, 16}."""
    cfg = _cfg("b", H, W, B, K, "bf16")
    fr = synth.gen_frames(cfg)
    out, _ = _run(cfg, fr, family)
    w = weights_for(cfg)
    for b in range(B):
        mx, mean = errs(out[b], oracle_full(cfg, w, fr, b))
        print(f"{family} {H}x{W} K={K} frame {b}: max {mx:.3e} mean {mean:.3e}")
        assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1]


@pytest.mark.parametrize("family", FAMILIES)
def test_mean_pool_and_c0_net_bf16(cuda_ok, family):
    cfg = synth.Config("m", 32, 64, 1, 4, 3, (16, 32, 64), 32, "bf16", pool="mean")
    fr = synth.gen_frames(cfg)
    out, _ = _run(cfg, fr, family)
    mx, mean = errs(out[0], oracle_full(cfg, weights_for(cfg), fr))
    assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1]


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("prec,K", [("bf16", 8), ("bf16", 16), ("fp32", 8)])
def test_permutation_garbage_bitwise(cuda_ok, family, prec, K):
    """P3/P4 on the GPU: permuting the valid slots and filling masked slots with NaN/Inf
    bit patterns gives a bitwise-identical output (table:OrderLoss P:666-679; R4, R5).
    K = 16 runs the T kernel's single-buffered layer-1 operand."""
    if prec == "fp32" and family == "tc":
        pytest.skip("fp32 check mode has only the FFMA family")
    rng = np.random.default_rng(5)
    cfg = _cfg("p", 32, 48, 1, K, prec)
    fr = synth.gen_frames(cfg)
    out, net = _run(cfg, fr, family)
    tb = fr.tbuf.copy()
    n = fr.tcount[0]
    garbage = (np.array([0x7FC0, 0x7F80, 0xFF80, 0xFFFF], np.uint16) if prec == "bf16"
               else np.array([np.nan, np.inf, -np.inf, 3e38], np.float32))
    for y in range(32):
        for x in range(48):
            m = int(n[y, x])
            tb[0, y, x, :m] = fr.tbuf[0, y, x, rng.permutation(m)]
            tb[0, y, x, m:] = rng.choice(garbage, size=(K - m, 11))
    fr2 = synth.Frames(fr.gbuf, fr.direct, tb, fr.tcount, prec)
    out2, _ = _run(cfg, fr2, family, net)
    assert np.array_equal(out.view(np.uint32), out2.view(np.uint32))
    out3, _ = _run(cfg, fr, family, net)                       # run-to-run determinism
    assert np.array_equal(out.view(np.uint32), out3.view(np.uint32))


@pytest.mark.parametrize("family", FAMILIES)
def test_empty_and_full_counts(cuda_ok, family):
    """P5: n = 0 everywhere (the empty-set latent) and n = K everywhere, and n > K clamps."""
    cfg = _cfg("e", 32, 32, 1, 8, "bf16")
    fr = synth.gen_frames(cfg)
    w = weights_for(cfg)
    for fill in (0, 8, 255):
        fr2 = synth.Frames(fr.gbuf, fr.direct, fr.tbuf, np.full_like(fr.tcount, fill), "bf16")
        out, _ = _run(cfg, fr2, family)
        fr_ref = synth.Frames(fr.gbuf, fr.direct, fr.tbuf, np.full_like(fr.tcount, min(fill, 8)), "bf16")
        mx, mean = errs(out[0], oracle_full(cfg, w, fr_ref))
        assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1], (fill, mx)


def test_forward_host_chunked_equals_device(cuda_ok):
    """glassnet_forward_host pipelines chunks of <= 4 frames over copy streams: bitwise the
    whole-batch device forward (frames are independent, R21; T's count sort regroups pixels
    across the chunk boundary, which by construction changes no per-pixel result)."""
    import torch
    from synth import device
    cfg = _cfg("h", 96, 128, 6, 8, "bf16")
    net = net_for(cfg)
    g, d, t, n = device.alloc_and_fill(cfg)
    ref = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    hg, hd, ht, hn = (x.cpu().pin_memory() for x in (g, d, t, n))
    hout = torch.empty(ref.shape, dtype=torch.float32).pin_memory()
    net.forward_host(hg, hd, ht, hn, hout)
    assert torch.equal(hout, ref.cpu())
    net.close()


def test_workspace_independent_of_K(cuda_ok):
    """P12 (fig:MemUsage): the library's workspace does not grow with K."""
    sizes = []
    for K in (4, 8, 16):
        cfg = _cfg("k", 64, 64, 2, K, "bf16")
        net = net_for(cfg)
        sizes.append(net.workspace_bytes())
        net.close()
    assert sizes[0] == sizes[1] == sizes[2], sizes


def test_families_agree(cuda_ok):
    """The tensor-core and SIMT families compute the same function (both vs each other)."""
    cfg = _cfg("fa", 48, 128, 1, 8, "bf16")
    fr = synth.gen_frames(cfg)
    a, net = _run(cfg, fr, "tc")
    b, _ = _run(cfg, fr, "simt", net)
    assert np.abs(a - b).max() < 3e-2


# ------------------------------------------------------------------ full-frame parity
def _full_frame(cfg_name, frames, family="tc"):
    """Every pixel of the named frames vs the fp64 oracle (banded over the host cores; the
    band oracle is bitwise the full-frame oracle, test_window_oracle.py)."""
    import torch
    from synth import device
    cfg = synth.CONFIGS[cfg_name]
    net = net_for(cfg)
    net.set_kernel_family(family == "tc")
    mask = synth.disc_mask(1, cfg.height, cfg.width) if cfg.tcount_mode == "discs" else None
    g, d, t, n = device.alloc_and_fill(cfg, mask=mask)
    out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    w = weights_for(cfg)
    res = []
    for f in frames:
        fr = frames_from_device(g[f:f + 1], d[f:f + 1], t[f:f + 1], n[f:f + 1])
        ref = band_oracle(cfg, w, fr)
        mx, mean = errs(out[f].cpu().numpy(), ref)
        res.append((f, mx, mean))
        print(f"FULLFRAME {cfg_name} frame {f} ({cfg.width}x{cfg.height}, K={cfg.k_slots}, every pixel): "
              f"max abs {mx:.3e} mean abs {mean:.3e}")
    net.close()
    for f, mx, mean in res:
        assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1], (cfg_name, f, mx, mean)


def test_full_frame_c1(cuda_ok):
    _full_frame("c1", [0, 1, 2, 3])


def test_full_frame_c2(cuda_ok):
    _full_frame("c2", [0])


def test_full_frame_c3_frame0_in_bench_batch(cuda_ok):
    """configs[3] in the launch configuration bench.py times (batch 32): frame 0 and frame 31."""
    _full_frame("c3", [0, 31])


def test_full_frame_c4(cuda_ok):
    _full_frame("c4", [0])


def test_repeated_forwards_bitwise(cuda_ok):
    """Many back-to-back forwards (the T kernel's mbarrier pipeline across tiles, K = 8 double-
    and K = 16 single-buffered): every output bitwise equal to the first (S:572 run-to-run)."""
    import torch
    from synth import device
    for cfg, reps in ((_cfg("r8", 96, 272, 3, 8, "bf16"), 60), (_cfg("r16", 64, 136, 2, 16, "bf16"), 60)):
        net = net_for(cfg)
        g, d, t, n = device.alloc_and_fill(cfg)
        first = net.forward(g, d, t, n).clone()
        for _ in range(reps):
            out = net.forward(g, d, t, n)
            assert torch.equal(out, first)
        net.close()


def test_output_guard_bands(cuda_ok):
    """Out-of-bounds write check (compute-sanitizer is closed on this pool): the output tensor is a
    view into a larger buffer whose guard bands (before and after) hold a NaN pattern; after
    forwards of ragged shapes (T tiles past the last pixel, K = 3 / 8 / 16) the guards are intact."""
    import torch
    from synth import device
    for H, W, B, K in ((40, 136, 2, 8), (24, 72, 1, 16), (32, 48, 3, 3)):
        cfg = _cfg("g", H, W, B, K, "bf16")
        net = net_for(cfg)
        g, d, t, n = device.alloc_and_fill(cfg)
        G = 4096
        size = B * H * W * 3
        buf = torch.full((G + size + G,), float("nan"), dtype=torch.float32, device="cuda")
        buf.view(torch.int32)[:G] = 0x7FC01234
        buf.view(torch.int32)[G + size:] = 0x7FC04321
        out = buf[G:G + size].view(B, H, W, 3)
        for _ in range(3):
            net.forward(g, d, t, n, out)
        torch.cuda.synchronize()
        head, tail = buf.view(torch.int32)[:G], buf.view(torch.int32)[G + size:]
        assert bool((head == 0x7FC01234).all()) and bool((tail == 0x7FC04321).all()), (H, W, B, K)
        assert bool(torch.isfinite(out).all())
        net.close()


# ------------------------------------------------------------------ N1: sigma-conditioned h
@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("H,W,K,B", [(40, 136, 8, 2), (32, 72, 16, 1), (24, 48, 3, 1)])
def test_sigma_cond_bf16_parity(cuda_ok, family, H, W, K, B):
    """SURVEY §8(f) N1 (the paper's h(b_i, sigma), sigma = e0 at the pixel): both kernel
    families vs the sigma-conditioned oracle, bf16 tolerance."""
    cfg = _cfg("sg", H, W, B, K, "bf16", extra={"sigma_cond": True})
    fr = synth.gen_frames(cfg)
    out, _ = _run(cfg, fr, family)
    w = weights_for(cfg)
    for b in range(B):
        mx, mean = errs(out[b], oracle_full(cfg, w, fr, b))
        print(f"N1 {family} {H}x{W} K={K} frame {b}: max {mx:.3e} mean {mean:.3e}")
        assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1]


def test_sigma_cond_fp32_check_mode(cuda_ok):
    """N1 in the fp32 check mode (c0 network): max abs <= 1e-4 vs the oracle."""
    cfg = synth.Config("sg32", 64, 64, 1, 4, 3, (16, 32, 64), 32, "fp32", extra={"sigma_cond": True})
    fr = synth.gen_frames(cfg)
    out, _ = _run(cfg, fr)
    mx, _ = errs(out[0], oracle_full(cfg, weights_for(cfg), fr))
    print(f"N1 fp32: max {mx:.3e}")
    assert mx <= FP32_TOL


def test_sigma_cond_every_record_in_every_slot(cuda_ok):
    """N1 keeps bit-exact slot invariance: all K cyclic rotations of full pixels give bitwise the same
    psi (the sigma MMAs are the same for every slot of a pixel)."""
    import torch
    from synth import device
    K = 8
    cfg = _cfg("sgr", 128, 256, 2, K, "bf16", extra={"sigma_cond": True})
    net = net_for(cfg)
    g, d, t, n = device.alloc_and_fill(cfg, seed=5)
    n.fill_(K)
    net.forward(g, d, t, n)
    psi0 = net.debug_psi(cfg.batch).clone()
    for k in range(1, K):
        net.forward(g, d, torch.roll(t, shifts=k, dims=3).contiguous(), n)
        psi = net.debug_psi(cfg.batch)
        torch.cuda.synchronize()
        assert torch.equal(psi.view(torch.int32), psi0.view(torch.int32)), k
    net.close()


def test_full_frame_c1_sigma_cond(cuda_ok):
    """N1 at configs[1] size, every pixel of all 4 frames vs the banded oracle."""
    import torch
    from synth import device
    c = synth.CONFIGS["c1"]
    cfg = synth.Config("c1s", c.height, c.width, c.batch, c.k_slots, c.levels, c.widths, c.t_hidden, "bf16",
                       extra={"sigma_cond": True})
    net = net_for(cfg)
    g, d, t, n = device.alloc_and_fill(cfg)
    out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    w = weights_for(cfg)
    for f in range(cfg.batch):
        ref = band_oracle(cfg, w, frames_from_device(g[f:f + 1], d[f:f + 1], t[f:f + 1], n[f:f + 1]))
        mx, mean = errs(out[f].cpu().numpy(), ref)
        print(f"FULLFRAME N1 c1 frame {f}: max abs {mx:.3e} mean abs {mean:.3e}")
        assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1]
    net.close()
