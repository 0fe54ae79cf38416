"""Whole-forward time of configs[3] (32 frames) for the library named by GN_LIB (CUDA events around
10 back-to-back forwards after 3 warm-ups) plus the per-stage profile -- interleaved A/B of builds."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, make_dims  # noqa: E402
from synth import device  # noqa: E402

cfg = synth.CONFIGS["c3"]
B = cfg.batch
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=B))
g, d, t, n = device.alloc_and_fill(cfg, nframes=B)
out = torch.empty((B, cfg.height, cfg.width, 3), dtype=torch.float32, device="cuda")
for _ in range(3):
    net.forward(g, d, t, n, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    net.forward(g, d, t, n, out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
net.profile_begin(net.launches_per_forward(B) * 5 + 20)
for _ in range(5):
    net.forward(g, d, t, n, out)
st = net.profile_end()
print(os.path.basename(os.environ.get("GN_LIB", "libglassnet.so")), f"forward {ms:.3f} ms ({B * 1000 / ms:.0f} fps)",
      " ".join(f"{k} {v[0] / v[1]:.3f}" for k, v in st.items() if k in ("conv_F0", "conv_F1", "T_B_psi")))
