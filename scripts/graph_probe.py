"""Eager vs CUDA-graph replay of one ModuLoRA linear fwd+bwd (dev probe).

   python scripts/graph_probe.py ROWS COLS TOKENS [BITS] [RANK]
Prints one JSON line: eager and graph ms per fwd+bwd (L2 flushed between steps)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from scripts.sweep import graphed, layers_for, independent_layers_step, time_steps  # noqa: E402
from paper_2309_16119_b200 import modulora as M  # noqa: E402


def main():
    rows, cols, m = (int(v) for v in sys.argv[1:4])
    bits = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    r = int(sys.argv[5]) if len(sys.argv) > 5 else 8
    layers = layers_for([(rows, cols)] * 2, bits, r, M.MaterializationStrategy.RowMaterialize)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    fn = independent_layers_step(layers, m)
    out = {"shape": [rows, cols], "tokens": m, "env": {k: v for k, v in os.environ.items()
                                                       if k.startswith("MLRA_")}}
    out["eager_ms"] = time_steps(fn, flush, steps=20)
    out["graph_ms"] = time_steps(graphed(fn), flush, steps=20)
    out["eager_ms_2"] = time_steps(fn, flush, steps=20)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
