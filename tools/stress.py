"""Run many back-to-back forwards per config (deadlock / race smoke for the mbarrier pipelines);
prints the per-config count and the max abs difference between the first and last outputs
(must be 0: run-to-run determinism)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
from synth import device
from paper_2405_19056_b200 import GlassNet, make_dims
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for name in ("c3", "c4", "c1", "c2"):
    cfg = synth.CONFIGS[name]
    B = 1 if name == "c4" else cfg.batch
    w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
    net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels,
                                precision=cfg.precision, max_batch=B, pool=cfg.pool))
    g, d, t, n = device.alloc_and_fill(cfg, nframes=B, seed=3)
    first = net.forward(g, d, t, n).clone()
    t0 = time.time()
    out = None
    for i in range(N):
        out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    diff = (out - first).abs().max().item()
    print(f"{name}: {N} forwards in {time.time() - t0:.1f} s, max |last - first| = {diff}", flush=True)
    assert diff == 0.0
    net.close()
    del g, d, t, n, out, first
    torch.cuda.empty_cache()
