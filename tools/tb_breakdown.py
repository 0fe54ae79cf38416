"""Per-phase clock64 breakdown of one T-kernel chain (diagnostic build, -DGN_PROFILE_TB)."""
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
tiles, rounds = v[11], v[10]
names = {0: "superblock sort", 1: "tile prologue (loads, rank, A1/e0 writes)", 2: "prologue barrier", 3: "round: MMA wait",
         4: "round: epilogues", 5: "round: barrier", 6: "final MMA wait", 7: "epilogue 3 (phi, psi)", 8: "round: MMA issue (thread 0)", 15: "round: epilogue 2 (pool, overlapped)", 9: "tile total",
         12: "  prologue: loads (tcount+records)", 13: "tile-start MMA issue (thread 0)", 14: "  prologue: rank + A1 writes"}
print(f"tiles={tiles} rounds={rounds} rounds/tile={rounds / max(tiles, 1):.2f}")
for i, nm in names.items():
    print(f"{nm:45s} {v[i] / max(tiles, 1):10.0f} cyc/tile" + (f"  {v[i] / max(rounds, 1):8.0f} cyc/round" if i in (3, 4, 5, 8, 15) else ""))
