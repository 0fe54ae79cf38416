"""Row-tile sharding (reading R22).

gpu: the per-rank steps of glassnet_forward_sharded, emulated on one device with the halo
rows moved by device copies (glassnet_forward_sharded_local), must reproduce the
single-GPU forward bitwise for 2/3/4 ranks.  The NCCL transport itself needs >= 2 GPUs
(tools/sharded_nccl_check.py under torchrun; test_nccl_sharded_multi_gpu).

not gpu: the tile split and the halo-exchange pattern with real multi-process
communication (torch.distributed gloo, world_size 2): each rank runs the fp64 oracle on
its row tile extended by rows received from its neighbours, and the gathered rows equal
the full-frame oracle bitwise (P13 with real sends/receives).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth
from helpers import BF16_TOL, errs, net_for, oracle_full, to_torch, weights_for

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ----------------------------------------------------------------------------- gpu
@pytest.mark.gpu
@pytest.mark.parametrize("H,W,K,nranks", [(96, 272, 8, 2), (96, 272, 8, 3), (128, 256, 16, 4), (64, 136, 4, 2)])
def test_sharded_local_bitwise_equals_single(cuda_ok, H, W, K, nranks):
    import torch
    from paper_2405_19056_b200 import glassnet as gb
    cfg = synth.Config("sh", H, W, 1, K, 4, (32, 64, 128, 256), 64, "bf16")
    fr = synth.gen_frames(cfg)
    g, d, t, n = to_torch(fr)
    single = net_for(cfg)
    ref = single.forward(g, d, t, n)
    nets, tiles = [], []
    for r in range(nranks):
        r0, rows = gb.tile_rows(single.dims, nranks, r)
        nets.append(net_for(cfg))
        sl = slice(r0, r0 + rows)
        tiles.append((g[:, sl].contiguous(), d[:, sl].contiguous(), t[:, sl].contiguous(), n[:, sl].contiguous(),
                      torch.empty((1, rows, W, 3), dtype=torch.float32, device="cuda")))
    gb.forward_sharded_local(nets, tiles)
    torch.cuda.synchronize()
    out = torch.cat([tl[4] for tl in tiles], dim=1)
    a, b = ref.cpu().numpy(), out.cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), np.abs(a - b).max()
    mx, mean = errs(b[0], oracle_full(cfg, weights_for(cfg), fr))
    assert mx <= BF16_TOL[0] and mean <= BF16_TOL[1]


@pytest.mark.gpu
def test_sharded_c4_full_size_local(cuda_ok):
    """configs[4] (3840x2160, K=16) split into 4 row tiles, emulated on one device:
    bitwise equal to the single-GPU frame."""
    import torch
    from paper_2405_19056_b200 import glassnet as gb
    from synth import device
    cfg = synth.CONFIGS["c4"]
    g, d, t, n = device.alloc_and_fill(cfg)
    single = net_for(cfg)
    ref = single.forward(g, d, t, n)
    torch.cuda.synchronize()
    nets, tiles = [], []
    for r in range(4):
        r0, rows = gb.tile_rows(single.dims, 4, r)
        nets.append(net_for(cfg))
        sl = slice(r0, r0 + rows)
        tiles.append((g[:, sl].contiguous(), d[:, sl].contiguous(), t[:, sl].contiguous(), n[:, sl].contiguous(),
                      torch.empty((1, rows, cfg.width, 3), dtype=torch.float32, device="cuda")))
    gb.forward_sharded_local(nets, tiles)
    torch.cuda.synchronize()
    out = torch.cat([tl[4] for tl in tiles], dim=1)
    assert torch.equal(ref.view(torch.int32), out.view(torch.int32))


@pytest.mark.gpu
def test_nccl_sharded_multi_gpu(cuda_ok):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("NCCL row-tile sharding needs >= 2 GPUs (this box has 1)")
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "tools", "sharded_nccl_check.py")]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "BITWISE_OK" in res.stdout


# ----------------------------------------------------------------------------- cpu (gloo)
def _gloo_worker(rank, world, port, H, W, K, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        widths, h, L = (16, 32, 64), 32, 3
        u = 1 << (L - 1)
        U = H // u
        r0, r1 = U * rank // world * u, U * (rank + 1) // world * u     # glassnet_tile_rows' rule
        cfg = synth.Config("g", H, W, 1, K, L, widths, h, "fp32")
        own = synth.gen_frames(cfg, seed=5, rows=(r0, r1))               # this rank's tile only
        g, d, t, n = (torch.from_numpy(np.ascontiguousarray(a[0])) for a in own.as64())
        margin = 24                                                      # >= receptive field, multiple of u
        # halo exchange: send my first/last `margin` rows to the neighbours, receive theirs
        parts = {}
        for name, a in (("g", g), ("d", d), ("t", t), ("n", n.to(torch.float64))):
            top = torch.zeros((margin,) + tuple(a.shape[1:]), dtype=a.dtype)
            bot = torch.zeros_like(top)
            reqs = []
            if rank > 0:
                reqs.append(dist.isend(a[:margin].contiguous(), rank - 1))
                reqs.append(dist.irecv(top, rank - 1))
            if rank < world - 1:
                reqs.append(dist.isend(a[-margin:].contiguous(), rank + 1))
                reqs.append(dist.irecv(bot, rank + 1))
            for rq in reqs:
                rq.wait()
            pieces = ([top] if rank > 0 else []) + [a] + ([bot] if rank < world - 1 else [])
            parts[name] = torch.cat(pieces, 0).numpy()
        a0 = r0 - (margin if rank > 0 else 0)
        rows_ext = parts["g"].shape[0]
        dims = oracle.make_dims(rows_ext, W, K, widths, h)
        wts = synth.make_weights(widths, L, h).astype(np.float64)
        out = oracle.forward(dims, wts, parts["g"], parts["d"], parts["t"], parts["n"].astype(np.uint8))
        mine = torch.from_numpy(np.ascontiguousarray(out[r0 - a0:r1 - a0]))
        gathered = [torch.zeros((U * (k + 1) // world * u - U * k // world * u, W, 3), dtype=torch.float64)
                    for k in range(world)]
        if rank == 0:
            full = [mine] + [torch.zeros_like(gathered[k]) for k in range(1, world)]
            for k in range(1, world):
                dist.recv(full[k], k)
            q.put(torch.cat(full, 0).numpy())
        else:
            dist.send(mine, 0)
    finally:
        dist.destroy_process_group()


def test_gloo_row_tiles_with_halo_exchange_equal_full_frame():
    import multiprocessing as mp
    H, W, K, world = 64, 32, 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, H, W, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.Config("g", H, W, 1, K, 3, (16, 32, 64), 32, "fp32")
    full = oracle_full(cfg, synth.make_weights((16, 32, 64), 3, 32), synth.gen_frames(cfg, seed=5))
    assert np.array_equal(got, full)


def test_halo_bench_harness_gloo():
    """tools/halo_bench.py (the §8(e) halo microbenchmark) at world size 2 with gloo on CPU: the
    neighbour exchange pattern completes and each halo row holds the neighbour's data."""
    import json as _json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "tools/halo_bench.py", "--cpu",
           "--iters", "5", "--warmup", "2"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
    d = _json.loads(line)
    assert d["world"] == 2 and all(p["ok"] for p in d["phases"].values())
