"""torchrun check of glassnet_forward_sharded over NCCL (needs >= 2 GPUs).

  python -m torch.distributed.run --nnodes=1 --nproc-per-node=N --master-addr 127.0.0.1 \
      tools/sharded_nccl_check.py [--config c4] [--frame-rows R]

Each rank fills its own row tile with the seeded device generator, runs the collective
forward, and rank 0 compares the gathered tiles with its single-GPU forward of the
whole frame bitwise (reading R22).  Prints BITWISE_OK on success.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import synth
    from paper_2405_19056_b200 import glassnet as gb
    from synth import device

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--frame-rows", type=int, default=0)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[a.config]
    if a.frame_rows:
        cfg = synth.Config(cfg.name, a.frame_rows, cfg.width, 1, cfg.k_slots, cfg.levels, cfg.widths, cfg.t_hidden,
                           cfg.precision)
    w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, bf16_weights=True)
    dims = gb.make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=1)
    net = gb.GlassNet(w, dims, device=local)
    uid = [gb.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = gb.Comm(uid[0], world, rank)
    r0, rows = gb.tile_rows(dims, world, rank)
    g, d, t, n = device.alloc_and_fill(cfg, nframes=1, rows=(r0, r0 + rows))
    out = torch.empty((1, rows, cfg.width, 3), dtype=torch.float32, device="cuda")
    net.forward_sharded(comm, g, d, t, n, out)
    torch.cuda.synchronize()
    tiles = [torch.empty((1, gb.tile_rows(dims, world, k)[1], cfg.width, 3), dtype=torch.float32, device="cuda")
             for k in range(world)]
    if rank == 0:
        tiles[0].copy_(out)
        for k in range(1, world):
            dist.recv(tiles[k], k)
        G, D, T, N = device.alloc_and_fill(cfg, nframes=1)
        ref = net.forward(G, D, T, N)
        torch.cuda.synchronize()
        full = torch.cat(tiles, 1)
        ok = torch.equal(ref.view(torch.int32), full.view(torch.int32))
        print("BITWISE_OK" if ok else f"MISMATCH max {float((ref - full).abs().max())}", flush=True)
    else:
        dist.send(out, 0)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
