"""GPU parity of the N3 super-sampler S (include/glassnet.h glassnet_supersample; SURVEY.md §8(f)
N3; reading N3) against the fp64 oracle, element by element:
both kernel families, bf16 (tolerance of BASELINE.json north_star: max 3e-2 / mean 3e-3 on the
[0,1] output) and the fp32 check mode (1e-4); ragged tiles (hi-res widths not multiples of 128),
full frames at c2 size and sampled c3 frames; SPEC's identity example bitwise; the pipeline
glassnet_forward -> glassnet_supersample.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import BF16_TOL, FP32_TOL, errs, ss_band_oracle, to_torch

pytestmark = pytest.mark.gpu

C1NET = dict(levels=4, widths=(32, 64, 128, 256), t_hidden=64)
C0NET = dict(levels=3, widths=(16, 32, 64), t_hidden=32)


def _net(H, W, B, prec, netc, wss=None, seed=0, K=4):
    from paper_2405_19056_b200 import GlassNet, make_dims
    dims = make_dims(H, W, K, netc["widths"], netc["t_hidden"], netc["levels"], precision=prec, max_batch=B,
                     supersample=True)
    w = synth.make_weights(netc["widths"], netc["levels"], netc["t_hidden"], seed=seed, bf16_weights=prec == "bf16")
    s = netc["widths"][0]
    if wss is None:
        wss = synth.make_ss_weights(s, seed=seed, bf16_weights=prec == "bf16")
    return GlassNet(np.concatenate([w, wss]), dims), wss


def _inputs(H, W, B, prec, seed=5):
    import torch
    img = synth.gen_image(seed, B, H, W)
    g = synth.gen_gbuf_hi(seed + 1, B, 2 * H, 2 * W, prec)
    gt = torch.from_numpy(np.ascontiguousarray(g).view(np.int16)).view(torch.bfloat16) if prec == "bf16" \
        else torch.from_numpy(g)
    g64 = synth.bf16_bits_to_f32(g).astype(np.float64) if prec == "bf16" else g.astype(np.float64)
    return img, torch.from_numpy(img).cuda(), gt.cuda(), g64


def _ss(net, img_t, g_t):
    import torch
    out = net.supersample(img_t, g_t)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("family", ["tc", "simt"])
@pytest.mark.parametrize("H,W,B", [(48, 136, 2), (8, 8, 1), (24, 200, 1)])
def test_ss_bf16_parity(cuda_ok, family, H, W, B):
    net, wss = _net(H, W, B, "bf16", C1NET)
    net.set_kernel_family(family == "tc")
    img, img_t, g_t, g64 = _inputs(H, W, B, "bf16")
    out = _ss(net, img_t, g_t)
    for b in range(B):
        ref = oracle.supersample(32, wss.astype(np.float64), img[b].astype(np.float64), g64[b])
        mx, mn = errs(out[b], ref)
        print(f"S {family} {H}x{W} frame {b}: max {mx:.3e} mean {mn:.3e}")
        assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1], (mx, mn)
    net.close()


def test_ss_fp32_check_mode(cuda_ok):
    H, W = 32, 40
    net, wss = _net(H, W, 1, "fp32", C0NET)
    img, img_t, g_t, g64 = _inputs(H, W, 1, "fp32")
    out = _ss(net, img_t, g_t)
    ref = oracle.supersample(16, wss.astype(np.float64), img[0].astype(np.float64), g64[0])
    mx, _ = errs(out[0], ref)
    print(f"S fp32: max {mx:.3e}")
    assert mx <= FP32_TOL
    net.close()


@pytest.mark.parametrize("family", ["tc", "simt"])
def test_ss_identity_residual_bitwise(cuda_ok, family):
    """identity-initialised residual (S3 = 0) -> out = nearest-upsampled img exactly."""
    H, W = 16, 72
    s = 32
    wss = synth.make_ss_weights(s, bf16_weights=True)
    wss[wss.size - 3 * s - 3:] = 0.0
    net, _ = _net(H, W, 1, "bf16", C1NET, wss=wss)
    net.set_kernel_family(family == "tc")
    img, img_t, g_t, _ = _inputs(H, W, 1, "bf16")
    out = _ss(net, img_t, g_t)
    assert np.array_equal(out[0], np.repeat(np.repeat(img[0], 2, 0), 2, 1))
    net.close()


def test_ss_full_frame_c2_size(cuda_ok):
    """Every pixel of a 1440x2560 output (c2's 720x1280 frame super-sampled), tensor cores."""
    H, W = 720, 1280
    net, wss = _net(H, W, 1, "bf16", C1NET)
    img, img_t, g_t, g64 = _inputs(H, W, 1, "bf16", seed=9)
    out = _ss(net, img_t, g_t)
    ref = ss_band_oracle(32, wss.astype(np.float64), img[0].astype(np.float64), g64[0])
    mx, mn = errs(out[0], ref)
    print(f"S full frame 1440x2560: max {mx:.3e} mean {mn:.3e}")
    assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()


def test_ss_c3_batch_sampled_bands(cuda_ok):
    """c3 geometry (32 frames of 1080x1920 -> 2160x3840), the bench's launch configuration:
    frames 0 and 31, a band of 8 low-res rows at the top, middle and bottom of each."""
    import torch
    H, W, B = 1080, 1920, 32
    net, wss = _net(H, W, B, "bf16", C1NET)
    img = synth.gen_image(5, B, H, W)
    img_t = torch.from_numpy(img).cuda()
    from synth import device
    hi = synth.Config("hi", 2 * H, 2 * W, B, 1, 4, C1NET["widths"], 64, "bf16")
    g_t, d_t, t_t, n_t = device.alloc_and_fill(hi, seed=6)
    del d_t, t_t, n_t
    out = net.supersample(img_t, g_t)
    torch.cuda.synchronize()
    w64 = wss.astype(np.float64)
    for b in (0, B - 1):
        for r0 in (0, H // 2 - 4, H - 8):
            a, e = max(0, r0 - 1), min(H, r0 + 9)
            g = synth.gen_frames(hi, seed=6, frame0=b, nframes=1, rows=(2 * a, 2 * e)).gbuf
            g64 = synth.bf16_bits_to_f32(g).astype(np.float64)[0]
            ref = oracle.supersample(32, w64, img[b, a:e].astype(np.float64), g64)[2 * (r0 - a):2 * (r0 - a) + 16]
            got = out[b, 2 * r0:2 * r0 + 16].cpu().numpy()
            mx, mn = errs(got, ref)
            print(f"S c3 frame {b} rows {r0}..{r0 + 8}: max {mx:.3e} mean {mn:.3e}")
            assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()


def test_forward_then_supersample(cuda_ok):
    """The paper's real-time pipeline: GlassNet's image, then S at x2, one handle."""
    import torch
    H, W = 32, 64
    cfg = synth.Config("p", H, W, 1, 8, 4, C1NET["widths"], 64, "bf16")
    net, wss = _net(H, W, 1, "bf16", C1NET, K=8)
    fr = synth.gen_frames(cfg, seed=2)
    g, d, t, n = to_torch(fr)
    img_t = net.forward(g, d, t, n)
    _, _, g_t, g64 = _inputs(H, W, 1, "bf16", seed=3)
    out = _ss(net, img_t, g_t)
    ref = oracle.supersample(32, wss.astype(np.float64), img_t.cpu().numpy()[0].astype(np.float64), g64[0])
    mx, mn = errs(out[0], ref)
    assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()


def test_ss_output_guard_bands_and_rerun_bitwise(cuda_ok):
    """Hazard check (compute-sanitizer is closed on this pool, profiles/r2_hazard_checks.md): S's
    epilogue writes exactly out_hi -- NaN guard bands before and after it stay untouched on a
    ragged frame (hi-res width 272 = 2 x 128 + 16) -- and 20 reruns give the same bits."""
    import torch
    H, W, B = 24, 136, 2
    net, _ = _net(H, W, B, "bf16", C1NET)
    img, img_t, g_t, _ = _inputs(H, W, B, "bf16")
    n = B * 2 * H * 2 * W * 3
    G = 4096
    buf = torch.full((n + 2 * G,), float("nan"), device="cuda")
    out = buf[G:G + n].view(B, 2 * H, 2 * W, 3)
    net.supersample(img_t, g_t, out)
    torch.cuda.synchronize()
    first = out.cpu().numpy().copy()
    assert torch.isnan(buf[:G]).all() and torch.isnan(buf[G + n:]).all()
    assert not np.isnan(first).any()
    for _ in range(20):
        net.supersample(img_t, g_t, out)
    torch.cuda.synchronize()
    assert np.array_equal(first.view(np.uint32), out.cpu().numpy().view(np.uint32))
    net.close()
