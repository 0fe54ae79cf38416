"""Bit-exact slot-permutation invariance of the tensor-core T path at scale (reading R5;
table:OrderLoss P:666-679 "identical rendering results"; BASELINE.json north_star
"bit-identical across layer permutations").

The T kernel puts every record in its own K=16 window, so a record's layer-1/layer-2 results
cannot depend on its slot, and the pool is an exact integer sum.  These tests check that
claim where round 1's could not: every record visits EVERY slot position (all K cyclic
rotations of a full pixel) over >= 10^6 pixels, comparing psi (the only place tau reaches
memory; glassnet_debug_psi) and the output bitwise; and random permutations of the valid
prefix with NaN/Inf garbage in masked slots on the full configs[3] batch and configs[4].
"""
import numpy as np
import pytest

import synth
from helpers import net_for

pytestmark = pytest.mark.gpu

C1NET = dict(levels=4, widths=(32, 64, 128, 256), t_hidden=64)
GARBAGE = np.array([0x7FC0, 0x7F80, 0xFF80, 0xFFFF, 0x7F7F], np.uint16)   # NaN, +Inf, -Inf, NaN, max


def _cfg(name, H, W, B, K):
    return synth.Config(name, H, W, B, K, C1NET["levels"], C1NET["widths"], C1NET["t_hidden"], "bf16")


def _permute_valid(t, n, seed, garbage=True):
    """Per pixel: a random permutation of the valid prefix k < n; masked slots filled with
    NaN/Inf bit patterns (device, frame by frame to bound memory)."""
    import torch
    B, H, W, K, _ = t.shape
    gen = torch.Generator(device=t.device)
    gen.manual_seed(seed)
    out = torch.empty_like(t)
    slot = torch.arange(K, device=t.device)
    gb = torch.from_numpy(GARBAGE.view(np.int16)).to(t.device)
    for b in range(B):
        m = n[b].clamp(max=K).long().unsqueeze(-1)
        valid = slot < m
        keys = torch.where(valid, torch.rand((H, W, K), generator=gen, device=t.device), 2.0 + slot.float())
        idx = keys.argsort(dim=-1).unsqueeze(-1).expand(H, W, K, 11)
        tb = torch.gather(t[b], 2, idx)
        if garbage:
            pick = torch.randint(0, len(GARBAGE), (H, W, K, 11), generator=gen, device=t.device)
            bits = torch.where(valid.unsqueeze(-1), tb.view(torch.int16), gb[pick])
            tb = bits.view(torch.bfloat16)
        out[b] = tb
    return out


@pytest.mark.parametrize("K", [8, 16])
def test_every_record_in_every_slot_psi_bitwise(cuda_ok, K):
    """n = K everywhere; all K cyclic rotations of every pixel's records (each record visits
    each slot, including round 1's split-window slots 2, 5, 10, 13): psi and the output are
    bitwise identical, over 8 x 256 x 512 = 1.05 M pixels."""
    import torch
    from synth import device
    cfg = _cfg("rot", 256, 512, 8, K)
    net = net_for(cfg)
    g, d, t, n = device.alloc_and_fill(cfg, seed=3)
    n.fill_(K)
    out0 = net.forward(g, d, t, n).clone()
    psi0 = net.debug_psi(cfg.batch)
    torch.cuda.synchronize()
    assert torch.isfinite(psi0).all()
    for k in range(1, K):
        out = net.forward(g, d, torch.roll(t, shifts=k, dims=3).contiguous(), n)
        psi = net.debug_psi(cfg.batch)
        torch.cuda.synchronize()
        assert torch.equal(psi.view(torch.int32), psi0.view(torch.int32)), f"rotation {k}: psi differs"
        assert torch.equal(out.view(torch.int32), out0.view(torch.int32)), f"rotation {k}: output differs"
    net.close()


def _full_perm(cfg_name, seeds):
    import torch
    from synth import device
    cfg = synth.CONFIGS[cfg_name]
    net = net_for(cfg)
    g, d, t, n = device.alloc_and_fill(cfg)
    out0 = net.forward(g, d, t, n).clone()
    psi0 = net.debug_psi(cfg.batch)
    torch.cuda.synchronize()
    for s in seeds:
        t2 = _permute_valid(t, n, s)
        out = net.forward(g, d, t2, n)
        psi = net.debug_psi(cfg.batch)
        torch.cuda.synchronize()
        assert torch.equal(psi.view(torch.int32), psi0.view(torch.int32)), (cfg_name, s, "psi")
        assert torch.equal(out.view(torch.int32), out0.view(torch.int32)), (cfg_name, s, "out")
        del t2
    net.close()


def test_permutation_garbage_bitwise_c3_full_batch(cuda_ok):
    """configs[3] as bench.py runs it (32 x 1920 x 1080, K=8): 3 permutation seeds."""
    _full_perm("c3", [11, 12, 13])


def test_permutation_garbage_bitwise_c4(cuda_ok):
    """configs[4] (3840 x 2160, K=16): 3 permutation seeds."""
    _full_perm("c4", [21, 22, 23])
