"""GPU parity of N2, the positional encoding of every input (GLASSNET_FLAG_POSENC(L); SURVEY.md
§8(f) N2, §3.4; reading N2) against the fp64
oracle: the tensor-core family (gamma(x) stored by k_prep_pe, F0 = the TMA implicit-GEMM conv
over 15(2L+1) -> 208 channels; T over 11(2L+1) encoded features per record on the SIMT kernel),
the SIMT family and the fp32 check mode; slot-permutation invariance bitwise; the row-tile
emulation bitwise equal to the full frame.
"""
import numpy as np
import pytest

import synth
from helpers import BF16_TOL, FP32_TOL, errs, net_for, oracle_full, to_torch, weights_for

pytestmark = pytest.mark.gpu

C1NET = dict(levels=4, widths=(32, 64, 128, 256), t_hidden=64)
C0NET = dict(levels=3, widths=(16, 32, 64), t_hidden=32)


def _cfg(H, W, B, K, prec, netc, pe_L, sigma=False):
    ex = {"pe_L": pe_L}
    if sigma:
        ex["sigma_cond"] = True
    return synth.Config("pe", H, W, B, K, netc["levels"], netc["widths"], netc["t_hidden"], prec, extra=ex)


def _run(cfg, fr, family=None):
    import torch
    net = net_for(cfg)
    if family is not None:
        net.set_kernel_family(family == "tc")
    g, d, t, n = to_torch(fr)
    out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    return out.cpu().numpy(), net


@pytest.mark.parametrize("family", ["tc", "simt"])
@pytest.mark.parametrize("H,W,K,pe_L,sigma", [(48, 136, 8, 6, False), (32, 64, 5, 3, False), (16, 264, 8, 6, True),
                                              (16, 136, 4, 1, False), (16, 136, 4, 10, False)])
def test_pe_bf16_parity(cuda_ok, family, H, W, K, pe_L, sigma):
    cfg = _cfg(H, W, 1, K, "bf16", C1NET, pe_L, sigma)
    fr = synth.gen_frames(cfg, seed=3)
    out, net = _run(cfg, fr, family)
    mx, mn = errs(out[0], oracle_full(cfg, weights_for(cfg), fr))
    print(f"PE {family} L={pe_L} sigma={sigma} {H}x{W}: max {mx:.3e} mean {mn:.3e}")
    assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()


@pytest.mark.parametrize("pe_L", [6, 10])
def test_pe_fp32_check_mode(cuda_ok, pe_L):
    cfg = _cfg(32, 48, 1, 4, "fp32", C0NET, pe_L)
    fr = synth.gen_frames(cfg, seed=4)
    out, net = _run(cfg, fr)
    mx, _ = errs(out[0], oracle_full(cfg, weights_for(cfg), fr))
    print(f"PE fp32: max {mx:.3e}")
    assert mx <= FP32_TOL
    net.close()


def test_pe_permutation_and_garbage_bitwise(cuda_ok):
    """Eq. eq:SymmetricNN with N2 (table:OrderLoss P:666-679): permuting each pixel's valid slots
    and filling masked slots with NaN leaves the output bitwise unchanged (tensor-core family)."""
    import torch
    cfg = _cfg(32, 136, 1, 8, "bf16", C1NET, 6)
    fr = synth.gen_frames(cfg, seed=6)
    a, net = _run(cfg, fr, "tc")
    t = fr.tbuf.copy()
    rng = np.random.default_rng(5)
    n = fr.tcount[0]
    for y in range(cfg.height):
        for x in range(cfg.width):
            m = int(n[y, x])
            t[0, y, x, :m] = t[0, y, x, rng.permutation(m)]
            t[0, y, x, m:] = 0x7FC0   # bf16 NaN
    fr2 = synth.Frames(fr.gbuf, fr.direct, t, fr.tcount, "bf16")
    g, d, tt, nn = to_torch(fr2)
    b = net.forward(g, d, tt, nn)
    torch.cuda.synchronize()
    assert np.array_equal(a.view(np.uint32), b.cpu().numpy().view(np.uint32))
    net.close()


def test_pe_row_tiles_bitwise(cuda_ok):
    """The row-tile path (gamma(x) with its halo rows exchanged before F0) equals the full frame."""
    import torch
    from paper_2405_19056_b200 import glassnet as gb
    cfg = _cfg(64, 136, 1, 8, "bf16", C1NET, 6)
    fr = synth.gen_frames(cfg)
    g, d, t, n = to_torch(fr)
    single = net_for(cfg)
    ref = single.forward(g, d, t, n)
    nets, tiles = [], []
    for r in range(2):
        r0, rows = gb.tile_rows(single.dims, 2, r)
        nets.append(net_for(cfg))
        sl = slice(r0, r0 + rows)
        tiles.append((g[:, sl].contiguous(), d[:, sl].contiguous(), t[:, sl].contiguous(), n[:, sl].contiguous(),
                      torch.empty((1, rows, cfg.width, 3), dtype=torch.float32, device="cuda")))
    gb.forward_sharded_local(nets, tiles)
    torch.cuda.synchronize()
    out = torch.cat([tl[4] for tl in tiles], dim=1)
    assert np.array_equal(ref.cpu().numpy().view(np.uint32), out.cpu().numpy().view(np.uint32))


def test_pe_c3_geometry_windows(cuda_ok):
    """N2 in the bench's launch configuration (c3 1920x1080, K=8, pe_L=6, tensor-core family; 4
    frames here): 16x32 windows at the corners and centre of frames 0 and 3 against the windowed
    oracle (margin 64; the encoding adds no receptive field)."""
    import torch
    from helpers import window_oracle
    from synth import device
    c3 = synth.CONFIGS["c3"]
    cfg = synth.Config("c3pe", c3.height, c3.width, 4, c3.k_slots, c3.levels, c3.widths, c3.t_hidden, "bf16",
                       extra={"pe_L": 6})
    net = net_for(cfg)
    g, d, t, n = device.alloc_and_fill(cfg, nframes=4, seed=1)
    out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    w = weights_for(cfg)
    H, W = cfg.height, cfg.width
    for b in (0, 3):
        for r0, c0 in ((0, 0), (H // 2, W // 2 - 16), (H - 16, W - 32)):
            rows, cols = (r0, r0 + 16), (c0, c0 + 32)
            ref = window_oracle(cfg, w, b, rows, cols, margin=64)
            mx, mn = errs(out[b, rows[0]:rows[1], cols[0]:cols[1]].cpu().numpy(), ref)
            print(f"PE c3 frame {b} window {rows}x{cols}: max {mx:.3e} mean {mn:.3e}")
            assert mx <= BF16_TOL[0] and mn <= BF16_TOL[1]
    net.close()
