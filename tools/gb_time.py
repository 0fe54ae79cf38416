"""A/B timing of conv variants (GN_LIB selects the library): per-stage CUDA-event times of the convs
in a c3 forward of 8 frames and of an 8-frame super-sample (ss_S1, ss_S2)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, make_dims  # noqa: E402
from synth import device  # noqa: E402

c3 = synth.CONFIGS["c3"]
H, W, K, B = c3.height, c3.width, c3.k_slots, 8
w = np.concatenate([synth.make_weights(c3.widths, 4, 64, bf16_weights=True), synth.make_ss_weights(32, bf16_weights=True)])
net = GlassNet(w, make_dims(H, W, K, c3.widths, 64, 4, max_batch=B, supersample=True))
g, d, t, n = device.alloc_and_fill(c3, nframes=B, seed=1)
hi = synth.Config("hi", 2 * H, 2 * W, B, 1, 4, c3.widths, 64, "bf16")
gh = device.alloc_and_fill(hi, nframes=B, seed=6)[0]
img = net.forward(g, d, t, n)
for _ in range(3):
    net.forward(g, d, t, n, img)
    o = net.supersample(img, gh)
torch.cuda.synchronize()
R = 10
net.profile_begin(40 * R)
for _ in range(R):
    net.forward(g, d, t, n, img)
    net.supersample(img, gh, o)
st = net.profile_end()
conv = sum(v[0] for k, v in st.items() if k.startswith("conv_")) / R
print(os.path.basename(os.environ.get("GN_LIB", "libglassnet.so")), f"convs {conv:.4f}",
      " ".join(f"{k} {v[0] / v[1]:.4f}" for k, v in st.items() if k.startswith(("conv_", "ss_", "up2")) or k == "T_B_psi"))
