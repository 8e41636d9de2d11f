"""Peer-to-peer copy-engine bandwidth probe (one process, all visible GPUs).

Measures cudaMemcpyAsync between GPUs issued by the destination (pull) or the source
(push), with 1..S streams splitting the bytes, and all GPUs pulling from all peers at
once (the all-to-all pattern).  Prints one JSON line per case.
"""
import itertools
import json
import sys

import torch


def timed(fn, reps=10):
    devs = range(torch.cuda.device_count())
    for d in devs:
        torch.cuda.synchronize(d)
    fn()
    for d in devs:
        torch.cuda.synchronize(d)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in devs]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in devs]
    import time
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    for d in devs:
        torch.cuda.synchronize(d)
    return (time.perf_counter() - t0) / reps


def main():
    n = torch.cuda.device_count()
    MB = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    nbytes = MB << 20
    bufs = [torch.empty(nbytes * n, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
    streams = {(d, k): torch.cuda.Stream(device=d) for d in range(n) for k in range(8)}
    for S in (1, 2, 4, 8):
        # pull 0 <- 1 with S streams on the destination
        def pull():
            chunk = nbytes // S
            for k in range(S):
                with torch.cuda.stream(streams[(0, k)]):
                    bufs[0][k * chunk:(k + 1) * chunk].copy_(bufs[1][k * chunk:(k + 1) * chunk], non_blocking=True)
        t = timed(pull)
        print(json.dumps({"case": "pull 0<-1", "streams": S, "GBps": nbytes / t / 1e9}), flush=True)

        def push():
            chunk = nbytes // S
            for k in range(S):
                with torch.cuda.stream(streams[(1, k)]):
                    bufs[0][k * chunk:(k + 1) * chunk].copy_(bufs[1][k * chunk:(k + 1) * chunk], non_blocking=True)
        t = timed(push)
        print(json.dumps({"case": "push 1->0 (issued on src)", "streams": S, "GBps": nbytes / t / 1e9}), flush=True)

        def a2a_pull():
            chunk = nbytes // S
            for d in range(n):
                for src in range(n):
                    if src == d:
                        continue
                    for k in range(S):
                        with torch.cuda.stream(streams[(d, (src + k) % 8)]):
                            off = src * nbytes + k * chunk
                            bufs[d][off:off + chunk].copy_(bufs[src][d * nbytes + k * chunk:d * nbytes + (k + 1) * chunk],
                                                           non_blocking=True)
        t = timed(a2a_pull)
        print(json.dumps({"case": f"all-to-all pull ({n} GPUs)", "streams_per_peer": S,
                          "GBps_per_gpu_in": (n - 1) * nbytes / t / 1e9}), flush=True)

        def a2a_push():
            chunk = nbytes // S
            for src in range(n):
                for d in range(n):
                    if src == d:
                        continue
                    for k in range(S):
                        with torch.cuda.stream(streams[(src, (d + k) % 8)]):
                            off = src * nbytes + k * chunk
                            bufs[d][off:off + chunk].copy_(bufs[src][d * nbytes + k * chunk:d * nbytes + (k + 1) * chunk],
                                                           non_blocking=True)
        t = timed(a2a_push)
        print(json.dumps({"case": f"all-to-all push ({n} GPUs)", "streams_per_peer": S,
                          "GBps_per_gpu_out": (n - 1) * nbytes / t / 1e9}), flush=True)


if __name__ == "__main__":
    main()
