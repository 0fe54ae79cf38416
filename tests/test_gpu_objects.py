"""GPU parity of N4, the object-major transparency path with a spatial h (glassnet_objects_begin /
add / finish; reading N4)
against the fp64 oracle (oracle.forward_objects): the tensor-core family (h's two 3x3 convs on
tcgen05, the second accumulating into the fixed-point latent in its epilogue), the SIMT family and
the fp32 check mode; object order and garbage outside the coverage bitwise; sampled windows at c3
geometry.  Synthetic objects: object k = slot k of a pixel-major frame, covered where k < n.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import BF16_TOL, FP32_TOL, errs, to_torch

pytestmark = pytest.mark.gpu

C1NET = dict(levels=4, widths=(32, 64, 128, 256), t_hidden=64)
C0NET = dict(levels=3, widths=(16, 32, 64), t_hidden=32)


def _setup(H, W, B, K, prec, netc, seed=3, pool="sum"):
    from paper_2405_19056_b200 import GlassNet, make_dims
    cfg = synth.Config("obj", H, W, B, K, netc["levels"], netc["widths"], netc["t_hidden"], prec, pool=pool)
    w = synth.make_weights(netc["widths"], netc["levels"], netc["t_hidden"], seed=0, bf16_weights=prec == "bf16",
                           objects=True)
    net = GlassNet(w, make_dims(H, W, K, netc["widths"], netc["t_hidden"], netc["levels"], precision=prec,
                                max_batch=B, objects=True, pool=pool))
    fr = synth.gen_frames(cfg, seed=seed)
    return cfg, w, net, fr


def _run(net, g, d, t, n, K, order=None):
    import torch
    B = g.shape[0]
    net.objects_begin(B)
    for k in (order or range(K)):
        net.objects_add(t[:, :, :, k, :].contiguous(), (n > k).to(torch.uint8).contiguous())
    out = net.objects_finish(g, d)
    torch.cuda.synchronize()
    return out


def _oracle(cfg, w, fr, b):
    g, d, t, n = fr.as64()
    dims = oracle.make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, objects=True,
                            pool=cfg.pool)
    objs, covs = oracle.objects_from_slots(t[b], n[b], cfg.k_slots)
    return oracle.forward_objects(dims, w.astype(np.float64), g[b], d[b], objs, covs)


@pytest.mark.parametrize("family", ["tc", "simt"])
@pytest.mark.parametrize("H,W,B,K,pool", [(48, 136, 2, 8, "sum"), (16, 264, 1, 5, "mean")])
def test_objects_bf16_parity(cuda_ok, family, H, W, B, K, pool):
    cfg, w, net, fr = _setup(H, W, B, K, "bf16", C1NET, pool=pool)
    net.set_kernel_family(family == "tc")
    out = _run(net, *to_torch(fr), K).cpu().numpy()
    for b in range(B):
        mx, mn = errs(out[b], _oracle(cfg, w, fr, b))
        print(f"N4 {family} {H}x{W} K={K} {pool} frame {b}: max {mx:.3e} mean {mn:.3e}")
        assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()


def test_objects_fp32_check_mode(cuda_ok):
    cfg, w, net, fr = _setup(32, 40, 1, 4, "fp32", C0NET)
    out = _run(net, *to_torch(fr), 4).cpu().numpy()
    mx, _ = errs(out[0], _oracle(cfg, w, fr, 0))
    print(f"N4 fp32: max {mx:.3e}")
    assert mx <= FP32_TOL
    net.close()


def test_objects_order_and_garbage_bitwise(cuda_ok):
    """P:764-775 / table:OrderLoss: the objects in any order, and NaN where an object does not
    cover, give the same bits (tensor-core family; exact fixed-point latent)."""
    import torch
    K = 6
    cfg, w, net, fr = _setup(32, 136, 1, K, "bf16", C1NET, seed=8)
    g, d, t, n = to_torch(fr)
    a = _run(net, g, d, t, n, K).cpu().numpy()
    b = _run(net, g, d, t, n, K, order=[4, 1, 5, 0, 3, 2]).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    t2 = t.clone()
    ks = torch.arange(K, device=t.device)[None, None, None, :, None]
    t2 = torch.where(ks >= n[..., None, None].long(), torch.full_like(t2, float("nan")), t2)
    c = _run(net, g, d, t2, n, K).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), c.view(np.uint32))
    net.close()


def test_objects_c3_geometry_windows(cuda_ok):
    """c3 geometry (1080x1920, K=8), a batch of 4 frames: 16x32 windows at the corners and centre of
    frames 0 and 3 against the windowed oracle (margin 64 >= the network's receptive field + h's 2 px)."""
    import torch
    from paper_2405_19056_b200 import GlassNet, make_dims
    from synth import device
    H, W, B, K = 1080, 1920, 4, 8
    c3 = synth.CONFIGS["c3"]
    w = synth.make_weights(c3.widths, c3.levels, c3.t_hidden, seed=0, bf16_weights=True, objects=True)
    net = GlassNet(w, make_dims(H, W, K, c3.widths, c3.t_hidden, c3.levels, max_batch=B, objects=True))
    g, d, t, n = device.alloc_and_fill(c3, nframes=B, seed=1)
    out = _run(net, g, d, t, n, K)
    u, margin = 8, 64
    w64 = w.astype(np.float64)
    for b in (0, B - 1):
        for r0, c0 in ((0, 0), (H // 2, W // 2 - 16), (H - 16, W - 32)):
            rows, cols = (r0, r0 + 16), (c0, c0 + 32)
            a_ = max(0, (rows[0] - margin) // u * u); b_ = min(H, -(-(rows[1] + margin) // u) * u)
            c_ = max(0, (cols[0] - margin) // u * u); e_ = min(W, -(-(cols[1] + margin) // u) * u)
            fr = synth.gen_frames(c3, seed=1, frame0=b, nframes=1, rows=(a_, b_), cols=(c_, e_))
            gg, dd, tt, nn = fr.as64()
            dims = oracle.make_dims(b_ - a_, e_ - c_, K, c3.widths, c3.t_hidden, c3.levels, objects=True)
            objs, covs = oracle.objects_from_slots(tt[0], nn[0], K)
            ref = oracle.forward_objects(dims, w64, gg[0], dd[0], objs, covs)
            ref = ref[rows[0] - a_:rows[1] - a_, cols[0] - c_:cols[1] - c_]
            got = out[b, rows[0]:rows[1], cols[0]:cols[1]].cpu().numpy()
            mx, mn = errs(got, ref)
            print(f"N4 c3 frame {b} window {rows}x{cols}: max {mx:.3e} mean {mn:.3e}")
            assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()


def test_objects_handle_refuses_pixel_major_forward(cuda_ok):
    from paper_2405_19056_b200 import glassnet as gb
    cfg, w, net, fr = _setup(16, 64, 1, 4, "bf16", C1NET)
    g, d, t, n = to_torch(fr)
    with pytest.raises(gb.GlassNetError, match="OBJECTS"):
        net.forward(g, d, t, n)
    net.close()


def test_objects_rerun_bitwise_and_guard_bands(cuda_ok):
    """Hazard check: 20 begin/add/finish sequences give the same bits (the latent's read-modify-
    write has one writer per pixel and launch), and the output's NaN guard bands stay untouched."""
    import torch
    K = 8
    cfg, w, net, fr = _setup(24, 136, 2, K, "bf16", C1NET, seed=9)
    g, d, t, n = to_torch(fr)
    objs = [t[:, :, :, k, :].contiguous() for k in range(K)]
    covs = [(n > k).to(torch.uint8).contiguous() for k in range(K)]
    N = 2 * 24 * 136 * 3
    G = 4096
    buf = torch.full((N + 2 * G,), float("nan"), device="cuda")
    out = buf[G:G + N].view(2, 24, 136, 3)

    def run():
        net.objects_begin(2)
        for k in range(K):
            net.objects_add(objs[k], covs[k])
        net.objects_finish(g, d, out)
        torch.cuda.synchronize()
        return out.cpu().numpy().copy()
    first = run()
    assert torch.isnan(buf[:G]).all() and torch.isnan(buf[G + N:]).all() and not np.isnan(first).any()
    for _ in range(20):
        assert np.array_equal(first.view(np.uint32), run().view(np.uint32))
    net.close()


@pytest.mark.parametrize("family", ["tc", "simt"])
def test_objects_empty_set(cuda_ok, family):
    """No object added (the empty set of Eq. eq:SymmetricNN): tau = 0 and n = 0 everywhere, as the
    oracle's t = 0 forward."""
    cfg, w, net, fr = _setup(16, 136, 1, 4, "bf16", C1NET, seed=10)
    net.set_kernel_family(family == "tc")
    g, d, t, n = to_torch(fr)
    net.objects_begin(1)
    out = net.objects_finish(g, d).cpu().numpy()
    g64, d64, _, _ = fr.as64()
    dims = oracle.make_dims(16, 136, 4, C1NET["widths"], C1NET["t_hidden"], 4, objects=True)
    ref = oracle.forward_objects(dims, w.astype(np.float64), g64[0], d64[0], [], [])
    mx, mn = errs(out[0], ref)
    assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()
