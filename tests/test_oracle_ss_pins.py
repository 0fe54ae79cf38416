"""Pins of the oracle's N3 super-sampler S (oracle.supersample, PAPER.md
§3.4; reading N3) against things other than itself:
SPEC's own identity example, a closed form for a constant residual, torch library routines
in fp64 (nearest interpolation + conv2d), and the receptive field of two 3x3 convolutions.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle
import synth


def _inputs(s, H, W, seed=3):
    w = synth.make_ss_weights(s, seed=seed).astype(np.float64)
    img = synth.gen_image(seed, 1, H, W)[0].astype(np.float64)
    g = synth.gen_gbuf_hi(seed + 1, 1, 2 * H, 2 * W, "fp32")[0].astype(np.float64)
    return w, img, g


def _zero_head(s, w, beta=(0.0, 0.0, 0.0)):
    w = w.copy()
    n = w.size
    w[n - 3 * s - 3:n - 3] = 0.0       # S3.W
    w[n - 3:] = beta                   # S3.b
    return w


@pytest.mark.parametrize("H,W", [(3, 5), (1, 1), (6, 4)])
def test_PS1_identity_residual_is_nearest_upsampling(H, W):
    """PS1 (SPEC S:439 'identity-initialized residual -> output = nearest-upsampled input'):
    with S3 = 0 every hi-res pixel (2i+a, 2j+b) equals img[i][j] exactly, output 2H x 2W."""
    s = 16
    w, img, g = _inputs(s, H, W)
    out = oracle.supersample(s, _zero_head(s, w), img, g)
    assert out.shape == (2 * H, 2 * W, 3)
    for a in (0, 1):
        for b in (0, 1):
            assert np.array_equal(out[a::2, b::2], img)


def test_PS2_constant_residual_closed_form():
    """PS2: S3.W = 0, S3.b = beta -> out = clamp(u + beta, 0, 1) (the head's bias and the clamp)."""
    s, H, W = 16, 4, 5
    w, img, g = _inputs(s, H, W)
    beta = (0.25, -0.5, 0.75)
    out = oracle.supersample(s, _zero_head(s, w, beta), img, g)
    u = np.repeat(np.repeat(img, 2, 0), 2, 1)
    exp = np.clip(u + np.array(beta), 0.0, 1.0)
    assert np.array_equal(out, exp)
    assert (out == 0.0).any() and (out == 1.0).any()      # both clamp ends exercised


@pytest.mark.parametrize("s,H,W,norm", [(16, 5, 7, True), (32, 4, 4, True), (16, 3, 6, False)])
def test_PS3_equals_torch_fp64_composition(s, H, W, norm):
    """PS3: torch fp64 library routines -- F.interpolate(mode='nearest', x2), F.conv2d (padding 1),
    ReLU, a 1x1 conv2d, clamp -- on the same inputs."""
    w, img, g = _inputs(s, H, W, seed=7)
    P = oracle.split_ss_weights(s, w)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.float64)
    im = t(img).permute(2, 0, 1)[None]
    u = Fnn.interpolate(im, scale_factor=2, mode="nearest")
    gg = t(g).permute(2, 0, 1)[None].clone()
    if norm:
        gg[:, 0:3] *= 0.125
        gg[:, 11] *= 0.0078125
    x = torch.cat([gg, u], 1)
    s1 = torch.relu(Fnn.conv2d(x, t(P["S1.W"]).permute(0, 3, 1, 2), t(P["S1.b"]), padding=1))
    s2 = torch.relu(Fnn.conv2d(s1, t(P["S2.W"]).permute(0, 3, 1, 2), t(P["S2.b"]), padding=1))
    r = Fnn.conv2d(s2, t(P["S3.W"])[:, :, None, None], t(P["S3.b"]))
    ref = torch.clamp(u + r, 0.0, 1.0)[0].permute(1, 2, 0).numpy()
    out = oracle.supersample(s, w, img, g, input_norm=norm)
    assert np.abs(out - ref).max() <= 1e-12


def test_PS4_receptive_field():
    """PS4: a change of img[i][j] reaches only hi-res pixels within 2 (two 3x3 convs) of its
    2x2 block -- catches a wrong nearest index (e.g. Y/2 on the wrong axis)."""
    s, H, W = 16, 6, 7
    w, img, g = _inputs(s, H, W)
    base = oracle.supersample(s, w, img, g)
    i, j = 2, 4
    img2 = img.copy()
    img2[i, j] = 1.0 - img2[i, j]
    diff = np.abs(oracle.supersample(s, w, img2, g) - base).max(axis=2) > 0
    ys, xs = np.nonzero(diff)
    assert ys.min() >= 2 * i - 2 and ys.max() <= 2 * i + 1 + 2
    assert xs.min() >= 2 * j - 2 and xs.max() <= 2 * j + 1 + 2
    assert diff[2 * i:2 * i + 2, 2 * j:2 * j + 2].all()    # the block itself always changes (u term)


def test_ss_weight_count():
    for s in (16, 32):
        assert oracle.ss_weight_count(s) == synth.make_ss_weights(s).size == 9 * 15 * s + s + 9 * s * s + s + 3 * s + 3


def test_ss_band_oracle_is_bitwise_the_full_frame():
    """The banded S oracle the full-size GPU parity tests use (one low-res row of margin) equals
    the whole-frame oracle bit for bit (S's receptive field is 2 hi-res pixels)."""
    from helpers import ss_band_oracle
    s, H, W = 16, 9, 6
    w, img, g = _inputs(s, H, W, seed=11)
    full = oracle.supersample(s, w, img, g)
    for band in (1, 2, 4):
        assert np.array_equal(ss_band_oracle(s, w, img, g, band=band, threads=2), full)


def test_ss_blob_layout_matches_library():
    """glassnet_weight_count with GLASSNET_FLAG_SUPERSAMPLE = the network's count + S's (s = c0)."""
    from paper_2405_19056_b200 import glassnet as gb
    for c in (synth.CONFIGS["c0"], synth.CONFIGS["c1"]):
        d0 = gb.make_dims(c.height, c.width, c.k_slots, c.widths, c.t_hidden, c.levels, precision=c.precision)
        d1 = gb.make_dims(c.height, c.width, c.k_slots, c.widths, c.t_hidden, c.levels, precision=c.precision,
                          supersample=True)
        assert gb.weight_count(d1) == gb.weight_count(d0) + oracle.ss_weight_count(c.widths[0])
