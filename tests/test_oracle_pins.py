"""Pins of the fp64 oracle against things other than itself.

Each test names the pin and the passage it follows.  None of these re-type the
oracle's loops: they use hand-derived golden values, a dense (Toeplitz) matrix
product, torch library routines in fp64, closed forms, exact invariants and
bitwise identities.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
rng = np.random.default_rng(1234)


# ----------------------------------------------------------------------------- P1
@pytest.mark.parametrize("pool", ["sum", "mean"])
def test_P1_T_pixel_hand_expanded(pool):
    """P1: single pixel, K=3, n=2, h=2, hand-expanded sums (Eq. eq:SymmetricNN)."""
    g = json.load(open(os.path.join(GOLDEN, "p1_T_pixel.json")))
    d = oracle.make_dims(1, 1, g["K"], (16, 32, 64), g["h"], pool=pool)
    tau = oracle.T_pixel(d, g["W1"], g["b1"], g["W2"], g["b2"], g["records"], g["n"])
    assert tau.tolist() == g["tau_sum" if pool == "sum" else "tau_mean"]
    tau0 = oracle.T_pixel(d, g["W1"], g["b1"], g["W2"], g["b2"], g["records"], 0)
    assert tau0.tolist() == g["tau_empty"]
    # n > K clamps to K (garbage slot 2 becomes valid -> differs)
    tau3 = oracle.T_pixel(d, g["W1"], g["b1"], g["W2"], g["b2"], g["records"], 200)
    assert tau3[-1] == 3.0


# ----------------------------------------------------------------------------- P2
def _toeplitz(Wt, H, Wd, stride):
    Cout, _, _, Cin = Wt.shape
    Ho, Wo = (H + stride - 1) // stride, (Wd + stride - 1) // stride
    M = np.zeros((Ho * Wo * Cout, H * Wd * Cin))
    for y in range(Ho):
        for x in range(Wo):
            for iy in range(H):
                ky = iy - stride * y + 1
                if not 0 <= ky < 3:
                    continue
                for ix in range(Wd):
                    kx = ix - stride * x + 1
                    if not 0 <= kx < 3:
                        continue
                    r0 = (y * Wo + x) * Cout
                    c0 = (iy * Wd + ix) * Cin
                    M[r0:r0 + Cout, c0:c0 + Cin] = Wt[:, ky, kx, :]
    return M


@pytest.mark.parametrize("stride,H,W", [(1, 5, 6), (2, 7, 6), (2, 6, 9), (1, 1, 1)])
def test_P2_conv_equals_dense_matrix(stride, H, W):
    """P2: direct conv == explicit dense matrix x vector (BJ north_star's brute-force list)."""
    Cin, Cout = 3, 4
    x = rng.standard_normal((H, W, Cin))
    Wt = rng.standard_normal((Cout, 3, 3, Cin))
    b = rng.standard_normal(Cout)
    got = oracle.conv3x3(x, Wt, b, stride, relu=False)
    M = _toeplitz(Wt, H, W, stride)
    ref = (M @ x.reshape(-1)).reshape(got.shape[0], got.shape[1], Cout) + b
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    # library routine: torch conv2d (cross-correlation, OIHW) in fp64
    t = Fnn.conv2d(torch.from_numpy(x).permute(2, 0, 1)[None], torch.from_numpy(Wt).permute(0, 3, 1, 2),
                   torch.from_numpy(b), stride=stride, padding=1)[0].permute(1, 2, 0).numpy()
    np.testing.assert_allclose(got, t, rtol=0, atol=1e-12)
    gotr = oracle.conv3x3(x, Wt, b, stride, relu=True)
    np.testing.assert_array_equal(gotr, np.where(got > 0, got, 0.0))


# ----------------------------------------------------------------------------- P7 / P8
def test_P7_identity_convs():
    """P7: 3x3 centre-tap identity -> ReLU(x + b) exactly (S:318 identity-conv idea)."""
    C = 5
    x = rng.standard_normal((6, 7, C))
    Wt = np.zeros((C, 3, 3, C))
    for c in range(C):
        Wt[c, 1, 1, c] = 1.0
    b = rng.standard_normal(C)
    np.testing.assert_array_equal(oracle.conv3x3(x, Wt, b, 1, True), np.maximum(x + b, 0.0))
    # a single off-centre tap is an exact shift (checks ky/kx orientation, no flip)
    Wt2 = np.zeros((C, 3, 3, C))
    for c in range(C):
        Wt2[c, 0, 2, c] = 1.0          # reads in[y-1][x+1]
    got = oracle.conv3x3(x, Wt2, np.zeros(C), 1, False)
    ref = np.zeros_like(x)
    ref[1:, :-1] = x[:-1, 1:]
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("H,W", [(8, 8), (7, 9), (2, 3)])
def test_P8_stride2_is_subsampled_stride1(H, W):
    """P8: s2 conv == s1 conv sampled at (2y, 2x), bitwise in fp64 (reading R10)."""
    x = rng.standard_normal((H, W, 3))
    Wt = rng.standard_normal((4, 3, 3, 3))
    b = rng.standard_normal(4)
    s1 = oracle.conv3x3(x, Wt, b, 1, True)
    s2 = oracle.conv3x3(x, Wt, b, 2, True)
    np.testing.assert_array_equal(s2, s1[::2, ::2])


# ----------------------------------------------------------------------------- P9
def test_P9_up2_constant_ramp_and_torch():
    """P9: bilinear x2, half-pixel, edge clamp (reading R14)."""
    v = np.full((3, 4, 2), 0.625)          # dyadic: every tap product is exact
    np.testing.assert_array_equal(oracle.up2(v, 6, 8), np.full((6, 8, 2), 0.625))
    np.testing.assert_allclose(oracle.up2(np.full((3, 4, 2), 0.7), 6, 8), 0.7, rtol=4e-16, atol=0)
    # separable ramp v[i][k] = a*i + c*k + b0 -> interior closed form a*(j/2-1/4) + c*(m/2-1/4) + b0
    a, c, b0 = 2.0, -4.0, 1.0
    h, w = 5, 6
    ii, kk = np.mgrid[0:h, 0:w]
    v = (a * ii + c * kk + b0)[..., None]
    up = oracle.up2(v, 2 * h, 2 * w)[..., 0]
    for j in range(1, 2 * h - 1):
        for m in range(1, 2 * w - 1):
            assert up[j, m] == a * (j / 2 - 0.25) + c * (m / 2 - 0.25) + b0
    assert up[0, 0] == v[0, 0, 0] and up[-1, -1] == v[-1, -1, 0]   # clamped corners
    # torch interpolate (bilinear, align_corners=False), odd crop included
    v = rng.standard_normal((7, 9, 3))
    t = Fnn.interpolate(torch.from_numpy(v).permute(2, 0, 1)[None], scale_factor=2, mode="bilinear",
                        align_corners=False)[0].permute(1, 2, 0).numpy()
    np.testing.assert_allclose(oracle.up2(v, 14, 18), t, rtol=0, atol=1e-15)
    np.testing.assert_allclose(oracle.up2(v, 13, 17), t[:13, :17], rtol=0, atol=1e-15)


# ----------------------------------------------------------------------------- helpers
def _frame(H, W, K, widths=(16, 32, 64), h=32, seed=1, precision="fp32"):
    cfg = synth.Config("t", H, W, 1, K, len(widths), tuple(widths), h, precision)
    fr = synth.gen_frames(cfg, seed=seed)
    g, d, t, n = fr.as64()
    wts = synth.make_weights(widths, len(widths), h, seed=0).astype(np.float64)
    dims = oracle.make_dims(H, W, K, widths, h)
    return dims, wts, g[0], d[0], t[0], n[0]


def torch_pe(x, L):
    """N2's gamma on the last axis with torch.sin/cos: channel c -> [v, sin(2^k pi v), cos(2^k pi v)]_k."""
    if L == 0:
        return x
    parts = [x[..., None]]
    for k in range(L):
        a = (2.0 ** k) * math.pi * x
        parts += [torch.sin(a)[..., None], torch.cos(a)[..., None]]
    return torch.cat(parts, -1).reshape(*x.shape[:-1], x.shape[-1] * (2 * L + 1))


def torch_forward(dims, wts, g, dr, tb, n):
    """Independent torch-fp64 composition of the same graph (P10)."""
    wd = {k: torch.from_numpy(v) for k, v in oracle.split_weights(dims, wts).items()}
    L, h = dims.L, dims.h
    c = list(dims.c)[:L]
    g, dr, tb = (torch.from_numpy(np.asarray(a, np.float64)) for a in (g, dr, tb))
    scale = torch.ones(12, dtype=torch.float64)
    scale[0:3] = 0.125
    scale[11] = 1 / 128
    x = torch_pe(torch.cat([g * scale, dr], -1), dims.pe_L).permute(2, 0, 1)[None]
    conv = lambda t, name, s: Fnn.relu(Fnn.conv2d(t, wd[name + ".W"].permute(0, 3, 1, 2), wd[name + ".b"],
                                                  stride=s, padding=1))
    e = [conv(x, "F0", 1)]
    for l in range(1, L):
        e.append(conv(e[-1], f"F{l}", 2))
    rs = torch.ones(11, dtype=torch.float64)
    rs[7] = 1 / 128
    rec = torch_pe(tb * rs, dims.pe_L)
    if dims.sigma_cond:   # N1: h's input is [record ; e0 at the pixel]
        sig = e[0][0].permute(1, 2, 0)[:, :, None, :].expand(-1, -1, dims.K, -1)
        rec = torch.cat([rec, sig], -1)
    m = torch.from_numpy(np.minimum(n.astype(np.int64), dims.K))
    mask = torch.arange(dims.K)[None, None, :] < m[..., None]
    a1 = Fnn.relu(rec @ wd["T1.W"].T + wd["T1.b"])
    a2 = Fnn.relu(a1 @ wd["T2.W"].T + wd["T2.b"])
    a2 = torch.where(mask[..., None], a2, torch.zeros((), dtype=torch.float64))
    tau = torch.cat([a2.sum(-2), m[..., None].double()], -1)
    phi = Fnn.relu(torch.cat([e[0][0].permute(1, 2, 0), tau], -1) @ wd["B.W"].T + wd["B.b"])
    dcur = e[L - 1]
    for l in range(L - 1, 0, -1):
        y = conv(dcur, f"R{l}", 1)
        up = Fnn.interpolate(y, scale_factor=2, mode="bilinear", align_corners=False)
        skip = e[l - 1] if l - 1 >= 1 else phi.permute(2, 0, 1)[None]
        dcur = up[:, :, :skip.shape[2], :skip.shape[3]] + skip
    logits = torch.cat([dcur[0].permute(1, 2, 0), dr], -1) @ wd["O.W"].T + wd["O.b"]
    return torch.sigmoid(logits).numpy(), tau.numpy()


# ----------------------------------------------------------------------------- P10
@pytest.mark.parametrize("H,W,K,widths,h", [(20, 24, 4, (16, 32, 64), 32), (13, 11, 3, (16, 32, 64), 32),
                                              (16, 24, 8, (16, 16, 32, 32), 16)])
def test_P10_forward_equals_torch_composition(H, W, K, widths, h):
    """P10: the whole oracle forward == an independent torch-fp64 composition (<= 1e-12)."""
    dims, wts, g, dr, tb, n = _frame(H, W, K, widths, h)
    out, dump = oracle.forward(dims, wts, g, dr, tb, n, dump=True)
    ref, tau = torch_forward(dims, wts, g, dr, tb, n)
    np.testing.assert_allclose(dump["tau"], tau, rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)
    assert 0.02 < out.std() and out.min() > 0 and out.max() < 1   # not saturated (R9)


# ----------------------------------------------------------------------------- P3-P6
def test_P3_P4_P5_permutation_garbage_empty():
    """P3 permutation of valid slots (table:OrderLoss P:666-679) -> bitwise equal;
    P4 NaN/Inf garbage in masked slots -> bitwise equal (reading R4);
    P5 n = 0 -> empty-set latent."""
    dims, wts, g, dr, tb, n = _frame(16, 16, 4)
    out, dump = oracle.forward(dims, wts, g, dr, tb, n, dump=True)
    tbp = tb.copy()
    for y in range(16):
        for x in range(16):
            m = min(int(n[y, x]), 4)
            perm = rng.permutation(m)
            tbp[y, x, :m] = tb[y, x, perm]
            tbp[y, x, m:] = rng.choice([np.nan, np.inf, -np.inf, 1e300], size=(4 - m, 11))
    outp, dumpp = oracle.forward(dims, wts, g, dr, tbp, n, dump=True)
    assert np.array_equal(out.view(np.uint64), outp.view(np.uint64))
    assert np.array_equal(dump["tau"].view(np.uint64), dumpp["tau"].view(np.uint64))
    zero = n == 0
    assert zero.any()
    assert np.all(dump["tau"][zero] == 0.0)


def test_P6_duplicate_additivity():
    """P6: two identical valid records -> sum part = 2 h(b) exactly."""
    dims = oracle.make_dims(1, 1, 4, (16, 32, 64), 32)
    wd = oracle.split_weights(dims, synth.make_weights((16, 32, 64), 3, 32).astype(np.float64))
    rec = rng.standard_normal((4, 11))
    one = oracle.T_pixel(dims, wd["T1.W"], wd["T1.b"], wd["T2.W"], wd["T2.b"], rec, 1)
    rec2 = rec.copy()
    rec2[1] = rec[0]
    two = oracle.T_pixel(dims, wd["T1.W"], wd["T1.b"], wd["T2.W"], wd["T2.b"], rec2, 2)
    assert np.array_equal(two[:-1], 2 * one[:-1]) and two[-1] == 2 and one[-1] == 1
    assert (one[:-1] > 0).any()


# ----------------------------------------------------------------------------- P11
def test_P11_homogeneity_bitwise():
    """P11: zero biases, n = 0 -> logits(2 x) == 2 logits(x) bitwise (no stray constants)."""
    dims, wts, g, dr, tb, n = _frame(16, 24, 4)
    wd = oracle.split_weights(dims, wts)
    w0 = wts.copy()
    p = 0
    for name, arr in wd.items():   # split_weights preserves blob order
        if name.endswith(".b"):
            w0[p:p + arr.size] = 0.0
        p += arr.size
    n0 = np.zeros_like(n)
    _, d1 = oracle.forward(dims, w0, g, dr, tb, n0, dump=True)
    _, d2 = oracle.forward(dims, w0, 2 * g, 2 * dr, tb, n0, dump=True)
    assert np.array_equal(d2["logits"], 2 * d1["logits"])
    assert np.abs(d1["logits"]).max() > 0.1


# ----------------------------------------------------------------------------- P13 / P14
def test_P13_row_tiles_with_halo_equal_full_frame():
    """P13: computing a row band from a halo-extended crop == full frame, bitwise
    (the semantics forward_sharded must reproduce, reading R22)."""
    H, W = 64, 24
    dims, wts, g, dr, tb, n = _frame(H, W, 4)
    full = oracle.forward(dims, wts, g, dr, tb, n)
    margin = 24                       # multiple of 2^(L-1) = 4, > receptive field
    r0, r1 = 24, 40
    a, b = r0 - margin, r1 + margin
    dsub = oracle.make_dims(b - a, W, 4, (16, 32, 64), 32)
    sub = oracle.forward(dsub, wts, g[a:b], dr[a:b], tb[a:b], n[a:b])
    assert np.array_equal(sub[r0 - a:r1 - a], full[r0:r1])


def test_P14_shift_equivariance():
    """P14: shifting the input by a multiple of 2^(L-1) shifts the output identically
    away from the borders (fp64 exact)."""
    H, W, s = 48, 48, 8
    dims, wts, g, dr, tb, n = _frame(H, W, 4)
    hh = 32
    d2 = oracle.make_dims(hh, hh, 4, (16, 32, 64), 32)
    A = oracle.forward(d2, wts, g[:hh, :hh], dr[:hh, :hh], tb[:hh, :hh], n[:hh, :hh])
    B = oracle.forward(d2, wts, g[s:s + hh, s:s + hh], dr[s:s + hh, s:s + hh], tb[s:s + hh, s:s + hh],
                       n[s:s + hh, s:s + hh])
    m = 12
    assert np.array_equal(A[s + m:hh - m, s + m:hh - m], B[m:hh - m - s, m:hh - m - s])


def test_weight_count_matches_survey():
    """§8(b): 50,700 (c0 net) and 787,340 (c1-c4 net)."""
    assert oracle.weight_count(oracle.make_dims(64, 64, 4, (16, 32, 64), 32)) == 50700
    assert oracle.weight_count(oracle.make_dims(64, 64, 8, (32, 64, 128, 256), 64)) == 787340
    assert synth.weight_count((16, 32, 64), 3, 32) == 50700


# ----------------------------------------------------------------------------- R5 range
def test_R5_pool_fixed_point_range():
    """Reading R5: the GPU pools each fragment's layer-2 output as a fixed-point
    integer round(a2 * 2^12) saturated at 2^23 (a2 < 2048), which makes the sum exact and
    order-independent.  Pin that the saturation never binds for the workloads: the oracle's
    per-fragment a2 (T_pixel with n = 1 returns one fragment's h(b)) over a sample of
    records drawn as in BJ.configs (K = 16, the c4 slot count; the c1-c4 network, seed-0
    He weights; records in bf16) stays far below 2048."""
    cfg = synth.Config("r5", 24, 32, 1, 16, 4, (32, 64, 128, 256), 64, "bf16")
    fr = synth.gen_frames(cfg, seed=3)
    _, _, t64, _ = fr.as64()
    wts = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True).astype(np.float64)
    d = oracle.make_dims(1, 1, 16, cfg.widths, cfg.t_hidden)
    w = oracle.split_weights(d, wts)
    recs = t64[0].reshape(-1, 16, 11)
    amax = 0.0
    for px in range(0, recs.shape[0], 3):
        for k in range(16):
            one = np.zeros((16, 11))
            one[0] = recs[px, k]
            tau = oracle.T_pixel(d, w["T1.W"], w["T1.b"], w["T2.W"], w["T2.b"], one, 1)
            amax = max(amax, float(tau[:64].max()))
    assert tau[64] == 1.0
    print(f"max per-fragment a2 over {recs.shape[0] // 3 * 16} records: {amax:.3f} (saturation 2048)")
    assert 0.0 < amax < 2048.0 / 16


# ----------------------------------------------------------------------------- N1: h(b, sigma)
def test_P1s_T_pixel_sigma_hand_expanded():
    """N1: the paper's literal h(b_i, sigma) (Eq. eq:SymmetricNN), layer 1
    over [record ; sigma]; a hand-expanded single pixel (tests/golden/p1s_T_pixel_sigma.json)."""
    g = json.load(open(os.path.join(GOLDEN, "p1s_T_pixel_sigma.json")))
    for pool, key in (("sum", "tau_sum"), ("mean", "tau_mean")):
        d = oracle.make_dims(1, 1, g["K"], (g["c0"], 4, 8), g["h"], pool=pool, input_norm=False, sigma_cond=True)
        tau = oracle.T_pixel(d, g["W1"], g["b1"], g["W2"], g["b2"], g["records"], 2, sigma=g["sigma"])
        assert list(tau) == g[key], (pool, tau)
    d = oracle.make_dims(1, 1, g["K"], (g["c0"], 4, 8), g["h"], input_norm=False, sigma_cond=True)
    assert list(oracle.T_pixel(d, g["W1"], g["b1"], g["W2"], g["b2"], g["records"], 1, sigma=g["sigma"])) == g["tau_n1"]
    assert list(oracle.T_pixel(d, g["W1"], g["b1"], g["W2"], g["b2"], g["records"], 2, sigma=[0, 0])) == g["tau_sigma0"]


def _sigma_blob(widths, h, levels, zero_sigma_cols=False, zero_record_cols=False, seed=0):
    w = synth.make_weights(widths, levels, h, seed=seed, sigma_cond=True).astype(np.float64)
    c0 = widths[0]
    T1 = w[:h * (11 + c0)].reshape(h, 11 + c0)
    if zero_sigma_cols:
        T1[:, 11:] = 0.0
    if zero_record_cols:
        T1[:, :11] = 0.0
    return w


def test_P15_sigma_cond_with_zero_sigma_weights_is_the_unconditioned_network():
    """N1 reduces to the pinned network: with the sigma columns of T1.W zero, the sigma-conditioned
    forward equals the unconditioned forward (same remaining weights) bitwise."""
    widths, h, L = (16, 32, 64), 32, 3
    cfg = synth.Config("s", 20, 24, 1, 4, L, widths, h, "fp32")
    fr = synth.gen_frames(cfg, seed=2)
    g, dr, tb, n = fr.as64()
    ws = _sigma_blob(widths, h, L, zero_sigma_cols=True)
    T1 = ws[:h * (11 + widths[0])].reshape(h, 11 + widths[0])
    wu = np.concatenate([T1[:, :11].reshape(-1), ws[h * (11 + widths[0]):]])
    ds = oracle.make_dims(20, 24, 4, widths, h, sigma_cond=True)
    du = oracle.make_dims(20, 24, 4, widths, h)
    assert oracle.weight_count(ds) == ws.size and oracle.weight_count(du) == wu.size
    a = oracle.forward(ds, ws, g[0], dr[0], tb[0], n[0])
    b = oracle.forward(du, wu, g[0], dr[0], tb[0], n[0])
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_P16_sigma_only_fragments():
    """N1: with the record columns of T1.W zero every valid fragment gives the same h(sigma), so a
    pixel with n = 2 pools exactly 2 h(sigma) whatever its records, and sigma changes tau."""
    widths, h = (16, 32, 64), 32
    w = _sigma_blob(widths, h, 3, zero_record_cols=True)
    dims = oracle.make_dims(1, 1, 4, widths, h, sigma_cond=True)
    wd = oracle.split_weights(dims, w)
    rng2 = np.random.default_rng(3)
    sigma = rng2.uniform(0, 2, 16)
    rec_a, rec_b = rng2.standard_normal((4, 11)), rng2.standard_normal((4, 11))
    one = oracle.T_pixel(dims, wd["T1.W"], wd["T1.b"], wd["T2.W"], wd["T2.b"], rec_a, 1, sigma=sigma)
    two = oracle.T_pixel(dims, wd["T1.W"], wd["T1.b"], wd["T2.W"], wd["T2.b"], rec_b, 2, sigma=sigma)
    assert np.array_equal(two[:h], 2.0 * one[:h]) and two[h] == 2.0
    other = oracle.T_pixel(dims, wd["T1.W"], wd["T1.b"], wd["T2.W"], wd["T2.b"], rec_a, 1, sigma=sigma + 0.5)
    assert not np.array_equal(other[:h], one[:h])


@pytest.mark.parametrize("H,W,K,widths,h", [(20, 24, 4, (16, 32, 64), 32), (16, 24, 8, (16, 16, 32, 32), 16)])
def test_P10s_sigma_forward_equals_torch_composition(H, W, K, widths, h):
    """P10 for N1: the sigma-conditioned oracle forward == an independent torch-fp64 composition in
    which h's layer 1 reads [record ; e0 at the pixel] (<= 1e-12)."""
    cfg = synth.Config("t", H, W, 1, K, len(widths), tuple(widths), h, "fp32")
    fr = synth.gen_frames(cfg, seed=4)
    g, dr, tb, n = fr.as64()
    wts = synth.make_weights(widths, len(widths), h, seed=0, sigma_cond=True).astype(np.float64)
    dims = oracle.make_dims(H, W, K, widths, h, sigma_cond=True)
    out, dump = oracle.forward(dims, wts, g[0], dr[0], tb[0], n[0], dump=True)
    ref, tau = torch_forward(dims, wts, g[0], dr[0], tb[0], n[0])
    np.testing.assert_allclose(dump["tau"], tau, rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)
