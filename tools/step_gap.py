"""Compare the CUDA-event time of K back-to-back forwards with the sum of the per-stage
profile (diagnostic: where do inter-stage / inter-step gaps go?)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
from synth import device as sdev
from paper_2405_19056_b200 import GlassNet, make_dims
cfg = synth.CONFIGS["c3"]
w = synth.make_weights(cfg.widths, cfg.levels, cfg.t_hidden, seed=0, bf16_weights=True)
net = GlassNet(w, make_dims(cfg.height, cfg.width, cfg.k_slots, cfg.widths, cfg.t_hidden, cfg.levels,
                            precision=cfg.precision, max_batch=cfg.batch, pool=cfg.pool))
g, d, t, n = sdev.alloc_and_fill(cfg, nframes=cfg.batch, seed=1)
out = torch.empty((cfg.batch, cfg.height, cfg.width, 3), dtype=torch.float32, device="cuda")
K = 10
for _ in range(3):
    net.forward(g, d, t, n, out)
torch.cuda.synchronize()
for trial in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for _ in range(K):
        net.forward(g, d, t, n, out)
    h1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"timed: {e0.elapsed_time(e1) / K:.3f} ms/step on the GPU; host launch {1000 * (h1 - h0) / K:.3f} ms/step")
    net.profile_begin(net.launches_per_forward(cfg.batch) * K + 2)
    for _ in range(K):
        net.forward(g, d, t, n, out)
    st = net.profile_end()
    print(f"profiled sum: {sum(v[0] for v in st.values()) / K:.3f} ms/step")
# per-forward events in an otherwise unprofiled loop
evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
evs[0].record()
for i in range(K):
    net.forward(g, d, t, n, out)
    evs[i + 1].record()
torch.cuda.synchronize()
print("per-forward ms:", " ".join(f"{evs[i].elapsed_time(evs[i + 1]):.2f}" for i in range(K)))
# the same with a stream synchronize between forwards
tt = []
for i in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); net.forward(g, d, t, n, out); b.record(); torch.cuda.synchronize()
    tt.append(a.elapsed_time(b))
print("isolated forward ms:", " ".join(f"{x:.2f}" for x in tt))
