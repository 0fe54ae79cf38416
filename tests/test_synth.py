"""The seeded generator module (synth/): tile invariance, distributions, bf16 rounding.

GPU twin check (device generator == numpy generator, bitwise) is marked gpu.
"""
import numpy as np
import pytest

import synth


def test_tile_invariance_bitwise():
    cfg = synth.Config("t", 40, 36, 2, 4, 3, (16, 32, 64), 32, "bf16")
    full = synth.gen_frames(cfg, seed=3)
    part = synth.gen_frames(cfg, seed=3, frame0=1, nframes=1, rows=(8, 24), cols=(4, 36))
    assert np.array_equal(full.gbuf[1, 8:24, 4:36], part.gbuf[0])
    assert np.array_equal(full.tbuf[1, 8:24, 4:36], part.tbuf[0])
    assert np.array_equal(full.tcount[1, 8:24, 4:36], part.tcount[0])
    assert np.array_equal(full.direct[1, 8:24, 4:36], part.direct[0])


def test_value_ranges_match_configs0():
    """BASELINE.json configs[0] distributions."""
    cfg = synth.Config("t", 64, 64, 1, 4, 3, (16, 32, 64), 32, "fp32")
    g, d, t, n = synth.gen_frames(cfg).as64()
    assert g[..., 0:3].min() >= -10 and g[..., 0:3].max() <= 10
    nrm = np.linalg.norm(g[..., 3:6], axis=-1)
    assert np.allclose(nrm, 1, atol=1e-6)
    assert g[..., 6:11].min() >= 0 and g[..., 6:11].max() <= 1
    assert g[..., 11].min() >= 0.1 and g[..., 11].max() <= 100
    ld = np.log(d)
    assert abs(ld.mean() + 1) < 0.05 and abs(ld.std() - 1) < 0.05      # lognormal(-1, 1)
    assert t[..., 6].min() >= 0.05 and t[..., 6].max() <= 0.95          # alpha
    assert t[..., 7].min() >= 0.1 and t[..., 7].max() <= 100            # depth
    assert np.allclose(np.linalg.norm(t[..., 0:3], axis=-1), 1, atol=1e-6)
    counts = np.bincount(n.ravel(), minlength=5)
    assert counts.min() > 0.15 * n.size and n.max() == 4                # n ~ U{0..4}


def test_exp_ieee_accuracy():
    x = np.linspace(-8, 6, 20001)
    assert np.abs(synth.exp_ieee(x) / np.exp(x) - 1).max() < 4e-16


def test_bf16_rounding_rne():
    x = np.array([1.0, 1.00390625, 1.005859375, 1.0078125 + 2 ** -9, -3.0], np.float64)
    # 1+2^-8 is a tie -> even (1.0); 1+1.5*2^-8 -> 1+2^-7; 1+2^-7+2^-9 -> 1+2^-7
    got = synth.round_to_bf16(x)
    assert got.tolist() == [1.0, 1.0, 1.0078125, 1.0078125, -3.0]


def test_disc_mask_coverage():
    m = synth.disc_mask(1, 72, 128)
    assert 0.7 <= m.mean() < 0.95
    cfg = synth.Config("c2s", 72, 128, 1, 8, 4, (32, 64, 128, 256), 64, "bf16", tcount_mode="discs")
    n = synth.gen_frames(cfg, mask=m).tcount[0]
    assert np.all((n == 0) == ~m) and n.max() == 8 and n[m].min() == 1


def test_weights_blob():
    w = synth.make_weights((32, 64, 128, 256), 4, 64, seed=0)
    assert w.dtype == np.dtype("<f4") and w.size == 787340
    w2 = synth.make_weights((32, 64, 128, 256), 4, 64, seed=0, bf16_weights=True)
    T1W = w2[:64 * 11]
    assert np.array_equal(T1W, synth.round_to_bf16(T1W))
    # He-normal scale of T2.W (fan_in 64): std ~ sqrt(2/64)
    T2W = w[64 * 11 + 64: 64 * 11 + 64 + 64 * 64]
    assert abs(T2W.std() / np.sqrt(2 / 64) - 1) < 0.08
