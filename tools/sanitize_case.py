"""One small forward+backward through the C ABI for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_case.py --config C1
    compute-sanitizer --tool racecheck python tools/sanitize_case.py --config C2 --tokens 256
    compute-sanitizer --tool synccheck python tools/sanitize_case.py --config C2 --tokens 256 --dropless

Prints SANITIZE_CASE OK when the results match the oracle (the sanitizer's own report
decides the run)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import lina_inputs as li  # noqa: E402
from tests.parity_util import compare, gpu_layer, oracle_layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--n-chunks", type=int, default=1)
    ap.add_argument("--dropless", action="store_true")
    a = ap.parse_args()
    cfg = li.CONFIGS[a.config]
    if a.tokens:
        cfg = li.with_tokens(cfg, a.tokens)
    Wg, W1, W2 = li.layer_weights(cfg, 1234)
    X, dY = li.layer_tokens(cfg, 1234, 0)
    C = 0 if a.dropless else None
    g = gpu_layer(cfg, a.n_chunks, X, Wg, W1, W2, dY, capacity=C)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY, capacity=cfg.tokens_per_rank if a.dropless else None)
    errs = compare(cfg, g, o)
    print("SANITIZE_CASE OK", a.config, cfg.tokens_per_rank, {k: f"{v:.2e}" for k, v in errs.items()}, flush=True)


if __name__ == "__main__":
    main()
