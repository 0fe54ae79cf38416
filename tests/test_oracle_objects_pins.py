"""Pins of the oracle's N4 object-major path (oracle.forward_objects, PAPER.md
P:257-258 per-object buffers, P:366-368 h a multi-layer CNN without down-sampling, P:764-775
streaming; reading N4) against the pinned pixel-major network (a reduction that holds
bit for bit), exact invariances, locality, and an independent torch-fp64 conv2d composition.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

import oracle
import synth

WIDTHS, H_T, L = (16, 32, 64), 32, 3


def _frame(H, W, K, seed=2):
    cfg = synth.Config("t", H, W, 1, K, L, WIDTHS, H_T, "fp32")
    g, d, t, n = synth.gen_frames(cfg, seed=seed).as64()
    return g[0], d[0], t[0], n[0]


def _obj_weights(seed=0):
    return synth.make_weights(WIDTHS, L, H_T, seed=seed, objects=True).astype(np.float64)


@pytest.mark.parametrize("pool", ["sum", "mean"])
def test_P17_centre_tap_objects_equal_the_pixel_major_network(pool):
    """With every off-centre tap of h's two 3x3 convs zero, the spatial h is the per-pixel MLP:
    the object-major forward over the slot decomposition (object k = slot k, covered where k < n)
    equals og_forward with the centre taps as T1.W / T2.W, bit for bit (Eq. eq:SymmetricNN)."""
    H, W, K = 14, 18, 4
    g, d, t, n = _frame(H, W, K)
    wo = _obj_weights()
    do = oracle.make_dims(H, W, K, WIDTHS, H_T, objects=True, pool=pool)
    dp = oracle.make_dims(H, W, K, WIDTHS, H_T, pool=pool)
    O = oracle.split_weights(do, wo)
    for name in ("T1.W", "T2.W"):
        c = O[name][:, 1, 1, :].copy()
        O[name][:] = 0.0
        O[name][:, 1, 1, :] = c
    wo2 = np.concatenate([v.reshape(-1) for v in O.values()])
    P = dict(O)
    P["T1.W"] = O["T1.W"][:, 1, 1, :]
    P["T2.W"] = O["T2.W"][:, 1, 1, :]
    wp = np.concatenate([v.reshape(-1) for v in P.values()])
    objs, covs = oracle.objects_from_slots(t, n, K)
    a = oracle.forward_objects(do, wo2, g, d, objs, covs)
    b = oracle.forward(dp, wp, g, d, t, n)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_PO1_object_order_and_PO2_garbage_outside_coverage_bitwise():
    """PO1 (table:OrderLoss P:666-679): any order of the objects -> the same bits;
    PO2 (R4 for objects): NaN / Inf where an object does not cover -> the same bits."""
    H, W, K = 12, 16, 5
    g, d, t, n = _frame(H, W, K, seed=3)
    w = _obj_weights()
    dims = oracle.make_dims(H, W, K, WIDTHS, H_T, objects=True)
    objs, covs = oracle.objects_from_slots(t, n, K)
    a = oracle.forward_objects(dims, w, g, d, objs, covs)
    perm = [3, 0, 4, 2, 1]
    b = oracle.forward_objects(dims, w, g, d, [objs[i] for i in perm], [covs[i] for i in perm])
    assert np.array_equal(a, b)
    junk = [np.where(c[..., None] > 0, o, np.nan) for o, c in zip(objs, covs)]
    junk[0][covs[0] == 0] = np.inf
    c2 = oracle.forward_objects(dims, w, g, d, junk, covs)
    assert np.array_equal(a, c2)


def test_PO3_locality_of_an_object():
    """Two 3x3 convs: an object's value at one pixel reaches tau only within Chebyshev distance 2."""
    H, W, K = 16, 16, 3
    g, d, t, n = _frame(H, W, K, seed=4)
    w = _obj_weights()
    dims = oracle.make_dims(H, W, K, WIDTHS, H_T, objects=True)
    objs = [np.ones((H, W, 11)) * 0.3 for _ in range(2)]
    covs = [np.ones((H, W), np.uint8) for _ in range(2)]
    _, base = oracle.forward_objects(dims, w, g, d, objs, covs, dump=True)
    objs[1] = objs[1].copy()
    objs[1][7, 9] = 2.0
    _, moved = oracle.forward_objects(dims, w, g, d, objs, covs, dump=True)
    diff = np.abs(moved["tau"] - base["tau"]).max(axis=2) > 0
    ys, xs = np.nonzero(diff)
    assert diff[7, 9] and ys.min() >= 5 and ys.max() <= 9 and xs.min() >= 7 and xs.max() <= 11


def test_PO4_tau_equals_torch_conv2d_sum():
    """tau = sum_i cover_i ReLU(conv(ReLU(conv(cover_i b_i')))) and n = sum_i cover_i, composed with
    torch fp64 F.conv2d (<= 1e-12)."""
    H, W, K = 10, 13, 4
    g, d, t, n = _frame(H, W, K, seed=5)
    w = _obj_weights()
    dims = oracle.make_dims(H, W, K, WIDTHS, H_T, objects=True)
    objs, covs = oracle.objects_from_slots(t, n, K)
    _, dump = oracle.forward_objects(dims, w, g, d, objs, covs, dump=True)
    Wd = {k: torch.from_numpy(v) for k, v in oracle.split_weights(dims, w).items()}
    tau = torch.zeros((H_T, H, W), dtype=torch.float64)
    cnt = torch.zeros((H, W), dtype=torch.float64)
    for o, c in zip(objs, covs):
        x = torch.from_numpy(o.copy())
        x[..., 7] = x[..., 7] / 128.0
        cm = torch.from_numpy(c.astype(np.float64))
        x = (x * cm[..., None]).permute(2, 0, 1)[None]
        h1 = Fnn.relu(Fnn.conv2d(x, Wd["T1.W"].permute(0, 3, 1, 2), Wd["T1.b"], padding=1))
        a2 = Fnn.relu(Fnn.conv2d(h1, Wd["T2.W"].permute(0, 3, 1, 2), Wd["T2.b"], padding=1))[0]
        tau += a2 * cm
        cnt += cm
    ref = torch.cat([tau.permute(1, 2, 0), cnt[..., None]], -1).numpy()
    np.testing.assert_allclose(dump["tau"], ref, rtol=1e-13, atol=1e-12)
