"""Pins of the oracle's N2 positional encoding (oracle.posenc and the forward with pe_L > 0;
SURVEY.md §8(f) N2, §3.4; reading N2) against
closed forms, SPEC's own examples, the unencoded network (a reduction that holds bit for bit)
and an independent torch-fp64 composition with torch.sin / torch.cos.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from test_oracle_pins import torch_forward


def test_PE1_spec_examples():
    """v = 0 -> (0, 0, 1, 0, 1, ...); v = 0.5, first frequency -> sin = 1, cos = 0."""
    L = 6
    z = oracle.posenc([0.0], L)
    assert z.tolist() == [0.0] + [0.0, 1.0] * L
    h = oracle.posenc([0.5], L)
    assert h[0] == 0.5 and h[1] == 1.0 and abs(h[2]) < 1e-16


def test_PE2_channel_count_and_blob():
    """c = 17, L = 6 -> 221 channels; the blob's F0 / T1 widths follow (15 -> 195, 11 -> 143)."""
    assert oracle.posenc(np.zeros(17), 6).size == 221
    widths, h = (16, 32, 64), 32
    d = oracle.make_dims(8, 8, 4, widths, h, pe_L=6)
    wd = oracle.split_weights(d, np.zeros(oracle.weight_count(d)))
    assert wd["F0.W"].shape == (16, 3, 3, 195) and wd["T1.W"].shape == (h, 143)
    assert oracle.weight_count(d) == synth.weight_count(widths, 3, h, pe_L=6)


def test_PE3_closed_forms_at_one_sixth():
    """gamma(1/6) at L = 4 against exact trigonometric values of pi/6 * 2^k (pi/6, pi/3, 2pi/3, 4pi/3)."""
    r3 = math.sqrt(3.0) / 2.0
    exp = [1 / 6, 0.5, r3, r3, 0.5, r3, -0.5, -r3, -0.5]
    np.testing.assert_allclose(oracle.posenc([1.0 / 6.0], 4), exp, rtol=0, atol=2e-15)
    # channel order: channel c occupies [c(2L+1), (c+1)(2L+1)) -- a second channel does not interleave
    two = oracle.posenc([1.0 / 6.0, 0.0], 4)
    np.testing.assert_allclose(two[:9], exp, rtol=0, atol=2e-15)
    assert two[9:].tolist() == [0.0] + [0.0, 1.0] * 4


def _pe_blob(widths, h, L, pe_L, seed=0):
    """A pe_L blob whose sin/cos columns (F0 and T1) are zero and whose v columns are the unencoded
    network's weights -> (pe blob, unencoded blob)."""
    wu = synth.make_weights(widths, L, h, seed=seed).astype(np.float64)
    du = oracle.make_dims(4, 4, 4, widths, h)
    dp = oracle.make_dims(4, 4, 4, widths, h, pe_L=pe_L)
    U = oracle.split_weights(du, wu)
    pe = 2 * pe_L + 1
    parts = []
    for name, arr in U.items():
        if name == "T1.W":
            a = np.zeros((h, 11 * pe)); a[:, ::pe] = arr; arr = a
        elif name == "F0.W":
            a = np.zeros(arr.shape[:3] + (15 * pe,)); a[..., ::pe] = arr; arr = a
        parts.append(arr.reshape(-1))
    wp = np.concatenate(parts)
    assert wp.size == oracle.weight_count(dp)
    return wp, wu


def test_P15pe_zero_frequency_weights_is_the_unencoded_network():
    """N2 reduces to the pinned network: with every sin/cos column of F0.W and T1.W zero, the encoded
    forward equals the unencoded forward bit for bit (catches a wrong column order or offset)."""
    widths, h = (16, 32, 64), 32
    cfg = synth.Config("s", 20, 24, 1, 4, 3, widths, h, "fp32")
    g, dr, tb, n = synth.gen_frames(cfg, seed=2).as64()
    wp, wu = _pe_blob(widths, h, 3, 6)
    a = oracle.forward(oracle.make_dims(20, 24, 4, widths, h, pe_L=6), wp, g[0], dr[0], tb[0], n[0])
    b = oracle.forward(oracle.make_dims(20, 24, 4, widths, h), wu, g[0], dr[0], tb[0], n[0])
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("H,W,K,widths,h,pe_L", [(20, 24, 4, (16, 32, 64), 32, 6), (16, 24, 8, (16, 16, 32, 32), 16, 3)])
def test_P10pe_forward_equals_torch_composition(H, W, K, widths, h, pe_L):
    """P10 for N2: the encoded oracle forward == a torch-fp64 composition with torch.sin/cos PE (<= 1e-12)."""
    cfg = synth.Config("t", H, W, 1, K, len(widths), tuple(widths), h, "fp32")
    g, dr, tb, n = synth.gen_frames(cfg, seed=4).as64()
    wts = synth.make_weights(widths, len(widths), h, seed=0, pe_L=pe_L).astype(np.float64)
    dims = oracle.make_dims(H, W, K, widths, h, pe_L=pe_L)
    out, dump = oracle.forward(dims, wts, g[0], dr[0], tb[0], n[0], dump=True)
    ref, tau = torch_forward(dims, wts, g[0], dr[0], tb[0], n[0])
    np.testing.assert_allclose(dump["tau"], tau, rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)
    assert 0.02 < out.std()


def test_pe_permutation_invariance():
    """Eq. eq:SymmetricNN with N2: permuting the valid slots leaves the output bitwise unchanged."""
    widths, h, K = (16, 32, 64), 32, 4
    cfg = synth.Config("t", 8, 8, 1, K, 3, widths, h, "fp32")
    g, dr, tb, n = synth.gen_frames(cfg, seed=5).as64()
    wts = synth.make_weights(widths, 3, h, seed=0, pe_L=4).astype(np.float64)
    dims = oracle.make_dims(8, 8, K, widths, h, pe_L=4)
    a = oracle.forward(dims, wts, g[0], dr[0], tb[0], n[0])
    tb2 = tb[0].copy()
    rng = np.random.default_rng(0)
    for y in range(8):
        for x in range(8):
            m = min(int(n[0][y, x]), K)
            tb2[y, x, :m] = tb2[y, x, rng.permutation(m)]
    b = oracle.forward(dims, wts, g[0], dr[0], tb2, n[0])
    assert np.array_equal(a, b)
