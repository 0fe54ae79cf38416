"""Time the T kernel's stage (forward of configs[3] x 8 frames, CUDA-event stage profile) for the
library named by GN_LIB (ablation / diagnostic builds)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
from paper_2405_19056_b200 import GlassNet, make_dims
from synth import device
cfg = synth.CONFIGS["c3"]
B = 8
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=B))
g, d, t, n = device.alloc_and_fill(cfg, nframes=B)
for _ in range(2):
    net.forward(g, d, t, n)
torch.cuda.synchronize()
net.profile_begin(net.launches_per_forward(B) * 5 + 2)
for _ in range(5):
    net.forward(g, d, t, n)
st = net.profile_end()
print(os.path.basename(os.environ.get("GN_LIB", "libglassnet.so")), "T_B_psi ms (8 frames):", round(st["T_B_psi"][0] / 5, 3))
