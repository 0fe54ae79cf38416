"""Per-phase clock64 breakdown of one T-kernel chain (diagnostic build, -DGN_PROFILE_TB):
thread 0 of chain 0 of CTA 0 (an epilogue thread)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GN_LIB"] = os.path.join(ROOT, "paper_2405_19056_b200", "libglassnet_prof.so")
import torch, synth
from synth import device
from paper_2405_19056_b200 import glassnet as gb
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
B = 1 if cfg.name == "c4" else cfg.batch
net = gb.GlassNet(synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, bf16_weights=True),
                  gb.make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=B))
g, d, t, n = device.alloc_and_fill(cfg, nframes=B)
L = gb.lib()
L.glassnet_debug_tb_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
net.forward(g, d, t, n); torch.cuda.synchronize()
L.glassnet_debug_tb_prof(buf, 1)
net.forward(g, d, t, n); torch.cuda.synchronize()
L.glassnet_debug_tb_prof(buf, 0)
v = list(buf)
tiles, rounds = v[11], v[10] - v[11]
names = {1: "E1 publish next tile (+ tile ids)", 3: "E1 slot: wait for L1 (d1)",
         4: "E1 slot: epilogue 1 (acc1 -> A2 in TMEM) + arrive", 9: "E1 tile total",
         12: "MMA slot: wait rdyA (E1)", 13: "MMA slot: wait free2 (E2)", 14: "MMA slot: issue L2", 15: "MMA slot: issue L1"}
print(f"tiles={tiles} rounds={rounds} rounds/tile={rounds / max(tiles, 1):.2f}")
for i, nm in names.items():
    print(f"{nm:50s} {v[i] / max(tiles, 1):8.0f} cyc/tile" + (f"  {v[i] / max(rounds, 1):6.0f} cyc/round" if i in (3, 4, 12, 13, 14, 15) else ""))
