"""Per-role clock64 breakdown of the T kernel (diagnostic build, -DGN_TB_PROF):
  python -c 'from paper_2405_19056_b200 import build as b; b.build_profile_lib()'
  python tools/tb_breakdown.py            # one c3 forward (32 frames) after a warm-up
Counters are one warp per role, summed over CTAs; printed per tile / per item per CTA."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GN_LIB"] = os.path.join(ROOT, "paper_2405_19056_b200", os.environ.get("TB_PROF_LIB", "libglassnet_prof.so"))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_19056_b200 import GlassNet, glassnet as gb, make_dims  # noqa: E402
from synth import device  # noqa: E402

cfg = synth.CONFIGS[os.environ.get("TB_CFG", "c3")]
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels,
                            max_batch=cfg.batch))
g, d, t, n = device.alloc_and_fill(cfg)
L = gb.lib()
L.glassnet_debug_tb_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 40)()
net.forward(g, d, t, n)
L.glassnet_debug_tb_prof(buf, 1)
net.forward(g, d, t, n)
torch.cuda.synchronize()
L.glassnet_debug_tb_prof(buf, 1)
v = list(buf)
ctas = 148
tiles, items = v[19], v[18]
names = {0: "A wait tileReady", 2: "A wait done2 (acc1 slot)", 20: "A layer1 issue+commit", 4: "A total",
         3: "C waits (tile, accB, tau)", 23: "C B issue", 31: "C total",
         1: "B wait rdyA", 11: "B wait free2", 21: "B layer2 issue+commit", 22: "B total",
         5: "loader wait metaFree", 6: "loader wait a1Free", 7: "loader total", 8: "loader bar.sync",
         30: "loader issue next tile", 25: "loader cp.async wait", 32: "loader meta + decode",
         33: "loader zero-fill", 34: "loader fence + hand-over", 26: "loader tile (all)",
         9: "E1 wait done1", 10: "E1 wait tileReady", 12: "E1 total", 16: "E1 item work",
         27: "psi total", 28: "psi wait doneB", 29: "psi wait tileReady",
         13: "E2 wait done2", 14: "E2 wait doneB (tau reuse)", 15: "E2 total", 17: "E2 item work", 24: "E2 tmem ld+wait"}
print(f"tiles {tiles} items {items} ({items / max(tiles, 1):.2f} items/tile); per CTA: {tiles / ctas:.0f} tiles")
for i, nm in names.items():
    print(f"  {nm:24s} {v[i] / ctas / 1e6:9.3f} Mcyc/CTA  {v[i] / max(tiles, 1):8.0f} cyc/tile  {v[i] / max(items, 1):8.0f} cyc/item")
