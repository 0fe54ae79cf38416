"""Hash of a c3 forward's output (2 frames, K=8) for the library named by GN_LIB: two builds of a
kernel variant must print the same digest (bitwise-equal outputs)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, make_dims  # noqa: E402
from synth import device  # noqa: E402

cfg = synth.CONFIGS["c3"]
B = 2
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=B))
g, d, t, n = device.alloc_and_fill(cfg, nframes=B, seed=3)
out = net.forward(g, d, t, n)
torch.cuda.synchronize()
print(os.path.basename(os.environ.get("GN_LIB", "libglassnet.so")), "out md5",
      hashlib.md5(out.cpu().numpy().tobytes()).hexdigest())
