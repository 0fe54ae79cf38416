"""Time the T kernel (stage T_B_psi) of configs[3] with a given library (diagnostic ablation
builds: python -c 'from paper_2405_19056_b200 import build as b; b.build_profile_lib(...)').
usage: python tools/tb_ablate.py libname.so [libname2.so ...]  (each in its own process)"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 2 or (len(sys.argv) == 2 and not sys.argv[1].startswith("--one=")):
    reps = int(os.environ.get("TB_REPS", "1"))
    res = {n: [] for n in sys.argv[1:]}
    for _ in range(reps):   # interleaved, so box drift hits every library alike
        for name in sys.argv[1:]:
            out = subprocess.run([sys.executable, __file__, "--one=" + name], capture_output=True, text=True, timeout=300)
            if out.returncode:
                print(f"{name:40s} FAILED {out.stderr.strip()[-300:]}")
                continue
            res[name].append(float(out.stdout.split()[1]))
    for name, v in res.items():
        v = sorted(v)
        if v:
            print(f"{name:40s} T_B_psi min {v[0]:.3f} median {v[len(v) // 2]:.3f} ms over {len(v)}")
    sys.exit(0)
name = sys.argv[1][6:]
sys.path.insert(0, ROOT)
os.environ["GN_LIB"] = os.path.join(ROOT, "paper_2405_19056_b200", name)
import torch, synth
from synth import device
from paper_2405_19056_b200 import glassnet as gb
cfg = synth.CONFIGS["c3"]
net = gb.GlassNet(synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, bf16_weights=True),
                  gb.make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels, max_batch=cfg.batch))
g, d, t, n = device.alloc_and_fill(cfg, nframes=cfg.batch)
for _ in range(2):
    net.forward(g, d, t, n)
torch.cuda.synchronize()
net.profile_begin(net.launches_per_forward(cfg.batch) * 5 + 2)
for _ in range(5):
    net.forward(g, d, t, n)
torch.cuda.synchronize()
st = net.profile_end()
print(f"T_B_psi {st['T_B_psi'][0] / 5:.3f} ms")
