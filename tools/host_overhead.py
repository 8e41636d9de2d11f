"""Host-side cost of one layer step (diagnostic): wall time of the forward / backward API
calls with the device idle before each call, and a cProfile of the Python side.
    python tools/host_overhead.py"""
import cProfile
import os
import pstats
import sys
import time

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
for _ in range(5):
    layer.forward(x, wg, w1, w2, out=y)
    layer.backward(dy, x, wg, w1, w2, dx, dwg, dw1, dw2)
torch.cuda.synchronize()
tf, tb = [], []
for _ in range(50):
    torch.cuda.synchronize()
    a = time.perf_counter()
    layer.forward(x, wg, w1, w2, out=y)
    b = time.perf_counter()
    layer.backward(dy, x, wg, w1, w2, dx, dwg, dw1, dw2)
    c = time.perf_counter()
    tf.append(b - a)
    tb.append(c - b)
tf.sort()
tb.sort()
print(f"host forward call  median {1e6 * tf[25]:.1f} us  min {1e6 * tf[0]:.1f}")
print(f"host backward call median {1e6 * tb[25]:.1f} us  min {1e6 * tb[0]:.1f}")
a = time.perf_counter()
for _ in range(50):
    torch.cuda.current_stream().cuda_stream
print(f"current_stream lookup {1e6 * (time.perf_counter() - a) / 50:.2f} us")
pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
for _ in range(20):
    layer.forward(x, wg, w1, w2, out=y)
    layer.backward(dy, x, wg, w1, w2, dx, dwg, dw1, dw2)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
comm.close()
