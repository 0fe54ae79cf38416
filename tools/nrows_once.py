"""One call of each §8(f) NEXT path at c3 geometry (4 frames) for an ncu capture of their kernels:
N3 supersample (k_conv_tc GB=2 / EPI=2), N4 objects (k_obj_prep, k_conv_tc EPI=3, k_b_psi),
N2 positional encoding (k_prep_pe, the 208-channel F0, k_tb_simt with PE).  Not a benchmark."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, make_dims  # noqa: E402
from synth import device  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
c3 = synth.CONFIGS["c3"]
H, W, K, B = c3.height, c3.width, c3.k_slots, 4
g, d, t, n = device.alloc_and_fill(c3, nframes=B, seed=1)
if which in ("all", "n3"):
    w = np.concatenate([synth.make_weights(c3.widths, 4, 64, bf16_weights=True), synth.make_ss_weights(32, bf16_weights=True)])
    net = GlassNet(w, make_dims(H, W, K, c3.widths, 64, 4, max_batch=B, supersample=True))
    img = net.forward(g, d, t, n)
    hi = synth.Config("hi", 2 * H, 2 * W, B, 1, 4, c3.widths, 64, "bf16")
    gh = device.alloc_and_fill(hi, nframes=B, seed=6)[0]
    net.supersample(img, gh)
    torch.cuda.synchronize()
    net.close()
    del gh
if which in ("all", "n4"):
    w = synth.make_weights(c3.widths, 4, 64, bf16_weights=True, objects=True)
    net = GlassNet(w, make_dims(H, W, K, c3.widths, 64, 4, max_batch=B, objects=True))
    net.objects_begin(B)
    for k in range(2):
        net.objects_add(t[:, :, :, k, :].contiguous(), (n > k).to(torch.uint8).contiguous())
    net.objects_finish(g, d)
    torch.cuda.synchronize()
    net.close()
if which in ("all", "n2"):
    w = synth.make_weights(c3.widths, 4, 64, bf16_weights=True, pe_L=6)
    net = GlassNet(w, make_dims(H, W, K, c3.widths, 64, 4, max_batch=1, pe_L=6))
    net.forward(g[:1], d[:1], t[:1], n[:1])
    torch.cuda.synchronize()
    net.close()
print("ok")
