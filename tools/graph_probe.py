"""CUDA-graph replay vs eager launch of one C2 fwd+bwd step at N=1 (diagnostic).
    python tools/graph_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lina_inputs as li  # noqa: E402
from paper_2210_17223_b200 import lina  # noqa: E402

cfg = li.CONFIGS["C2"]
dev = torch.device("cuda", 0)
comm = lina.Comm(1, 0, 0)
T, d, f, E, k = cfg.tokens_per_rank, cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k
Wg, W1, W2 = li.layer_weights(cfg, 0, "balanced")
X, dY = li.layer_tokens(cfg, 0, 0, "balanced")
wg = torch.from_numpy(Wg).to(dev)
w1 = torch.from_numpy(W1).to(torch.bfloat16).to(dev)
w2 = torch.from_numpy(W2).to(torch.bfloat16).to(dev)
x = torch.from_numpy(X).to(torch.bfloat16).to(dev)
dy = torch.from_numpy(dY).to(torch.bfloat16).to(dev)
layer = lina.MoELayer(comm, T, d, f, E, k, cfg.capacity(), 1, torch.bfloat16, dev)
y = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
dx, dwg, dw1, dw2 = torch.empty_like(x), torch.empty_like(wg), torch.empty_like(w1), torch.empty_like(w2)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()


def step():
    layer.forward(x, wg, w1, w2, out=y)
    layer.backward(dy, x, wg, w1, w2, dx, dwg, dw1, dw2)


with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.synchronize()
y_ref = y.clone()


def timed(fn, n=30):
    ts = []
    with torch.cuda.stream(s):
        for _ in range(n):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) for a, b in ts)
    return v[len(v) // 2]


print("eager median ms", timed(step))
print("graph median ms", timed(g.replay))
step()
torch.cuda.synchronize()
print("graph output matches eager:", bool(torch.equal(y, y_ref)))
