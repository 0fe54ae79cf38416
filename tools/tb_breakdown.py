"""Per-phase clock64 breakdown of one T-kernel chain (diagnostic build, -DGN_PROFILE_TB):
thread 0 of chain 0 of CTA 0 (an epilogue thread)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GN_LIB"] = os.path.join(ROOT, "paper_2405_19056_b200", os.environ.get("TB_PROF_LIB", "libglassnet_prof.so"))
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
buf = (ctypes.c_ulonglong * 32)()
net.forward(g, d, t, n); torch.cuda.synchronize()
L.glassnet_debug_tb_prof(buf, 1)
net.forward(g, d, t, n); torch.cuda.synchronize()
L.glassnet_debug_tb_prof(buf, 0)
v = list(buf)
tiles, rounds = v[11], v[10] - v[11]
names = {12: "E1 prologue: to the named barrier", 13: "E1 prologue: named barrier", 14: "E1 prologue: Kt, arrives",
         1: "E1 prologue (publish, e0, next records)", 3: "E1 slot: wait done1",
         4: "E1 slot: epilogue 1 + arrive", 6: "E1 wait doneF", 8: "E1 final", 9: "E1 tile total",
         16: "E2 wait tstart", 17: "E2 ring entry: wait done2", 18: "E2 slot: pool", 21: "E2 final (accB entry)",
         22: "E2 tile total (after tstart)",
         24: "MMA wait rdyC", 25: "MMA wait loaded", 26: "MMA L1(0) issue (+B if Kt=0)",
         27: "MMA slot: wait rdyA", 28: "MMA slot: wait free2", 29: "MMA slot: issue L2+L1+commits",
         30: "MMA slot: issueB (round 0)", 31: "MMA issueB: wait rdyF + e0"}
per_round = (3, 4, 17, 18, 27, 28, 29)
print(f"tiles={tiles} rounds={rounds} rounds/tile={rounds / max(tiles, 1):.2f}")
for i, nm in names.items():
    print(f"{nm:50s} {v[i] / max(tiles, 1):8.0f} cyc/tile" + (f"  {v[i] / max(rounds, 1):6.0f} cyc/round" if i in per_round else ""))
