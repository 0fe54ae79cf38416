"""Small forwards through every kernel family for compute-sanitizer (one tool per gpurun call):
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_run.py
bf16 tensor-core family (F0 from the G-buffer, stride-1/2 convs, streamed weights, the T kernel at
K = 3 / 8 / 16, up2add, output) at a c1-network frame of 64 x 256 (several T tiles, ragged); the
fp32 check mode (SIMT) at configs[0] (64 x 64, K = 4)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, make_dims  # noqa: E402
from synth import device  # noqa: E402

for name, H, W, B, K, widths, h, prec in (("tc K8", 64, 256, 2, 8, (32, 64, 128, 256), 64, "bf16"),
                                          ("tc K16", 64, 136, 1, 16, (32, 64, 128, 256), 64, "bf16"),
                                          ("tc K3", 32, 128, 1, 3, (32, 64, 128, 256), 64, "bf16"),
                                          ("simt c0", 64, 64, 1, 4, (16, 32, 64), 32, "fp32")):
    cfg = synth.Config("s", H, W, B, K, len(widths), widths, h, prec)
    w = synth.make_weights(widths, len(widths), h, seed=0, bf16_weights=prec == "bf16")
    net = GlassNet(w, make_dims(H, W, K, widths, h, len(widths), precision=prec, max_batch=B))
    g, d, t, n = device.alloc_and_fill(cfg, nframes=B)
    for _ in range(2):
        out = net.forward(g, d, t, n)
    torch.cuda.synchronize()
    print(name, "ok", float(out.mean()))
    net.close()
