"""configs[4] (3840x2160, K=16, one frame) in N row tiles, emulated on one GPU
(glassnet_forward_sharded_local: every rank's per-tile steps, halos by device copies): the time of
all N tiles back to back / N ~ one rank's compute (tiles differ by at most one 8-row unit), and a
prediction of the N-GPU frame time = max rank compute + halo exchanges.
  python tools/tile_times.py [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, glassnet as gb, make_dims  # noqa: E402
from synth import device  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = synth.CONFIGS["c4"]
H, W, K = cfg.height, cfg.width, cfg.k_slots
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
dims = make_dims(H, W, K, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=1)
g, d, t, n = device.alloc_and_fill(cfg, nframes=1)
# halo bytes one interior rank receives per frame: e0..e2 rows (stride-2 layers read 1 row above),
# x16 (F0), y/d rows of the decoder, z; every level's row is W/2^l * c_l * 2 bytes
c = cfg.widths
row_b = {"x16": W * 16 * 2}
for l in range(cfg.levels):
    row_b[f"e{l}"] = (W >> l) * c[l] * 2
res = {"config": "c4 3840x2160 K=16, one frame", "reps": reps, "N": {}}
t1 = None
for N in (1, 2, 4, 8):
    nets, tiles = [], []
    for r in range(N):
        r0, rows = gb.tile_rows(dims, N, r)
        nets.append(GlassNet(w, dims))
        sl = slice(r0, r0 + rows)
        tiles.append((g[:, sl].contiguous(), d[:, sl].contiguous(), t[:, sl].contiguous(), n[:, sl].contiguous(),
                      torch.empty((1, rows, W, 3), dtype=torch.float32, device="cuda"), rows))
    tt = [x[:5] for x in tiles]
    for _ in range(3):
        gb.forward_sharded_local(nets, tt)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        gb.forward_sharded_local(nets, tt)
    b.record()
    torch.cuda.synchronize()
    all_ms = a.elapsed_time(b) / reps
    max_rows = max(x[5] for x in tiles)
    rank_ms = all_ms * max_rows / H
    if N == 1:
        t1 = all_ms
    # exchange model: 10 grouped send/recv phases per frame (x16, e0..e3, y3, d2, y2, d1, z), each
    # ~15 us of NCCL latency on NVLink at these 0.1-0.5 MB sizes (bandwidth time < 1 us at 770 GB/s)
    exch_ms = 0.0 if N == 1 else 10 * 0.015
    pred = rank_ms + exch_ms
    # boundary rows first (the tile step list, GN_TILE_SPLIT policy): the exchanges of split producers
    # run beside their interior rows (counted hidden); the others stay exposed
    pol = int(os.environ.get("GN_TILE_SPLIT", "1"))
    nsplit = 0 if pol == 0 else (4 if pol == 1 else 9)
    pred_bf = rank_ms + (0.0 if N == 1 else (10 - nsplit) * 0.015)
    res["N"][str(N)] = {"all_tiles_ms": all_ms, "max_rank_rows": max_rows, "rank_compute_ms": rank_ms,
                        "exchange_model_ms": exch_ms, "predicted_frame_ms": pred,
                        "predicted_efficiency": t1 / (N * pred), "compute_only_efficiency": t1 / (N * rank_ms),
                        "predicted_frame_ms_boundary_first": pred_bf,
                        "predicted_efficiency_boundary_first": t1 / (N * pred_bf)}
    print(N, json.dumps(res["N"][str(N)]), flush=True)
    for x in nets:
        x.close()
    del nets, tiles, tt
    torch.cuda.empty_cache()
print(json.dumps(res))
