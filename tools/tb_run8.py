import sys, torch
sys.path.insert(0, '.')
import synth
from paper_2405_19056_b200 import GlassNet, make_dims
from synth import device
cfg = synth.CONFIGS["c3"]
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=8))
g, d, t, n = device.alloc_and_fill(cfg, nframes=8)
for _ in range(2):
    net.forward(g, d, t, n)
torch.cuda.synchronize()
print("ok")
