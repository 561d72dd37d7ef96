"""spmv_step (repr.cpp:193-237) on device operands: CUDA-event time of the
warp-per-unit kernel against its streaming roofline (4 B per col cell + 8 B
per row of x read once + 8 B per row of out written), per semiring."""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
g = ssb.gen_kronecker(a.scale, 16, 1)
r = ssb.build_slimsell(g, 32, g.num_vertices())
del g
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
x = torch.randint(0, 1 << 20, (r.n_padded,), dtype=torch.int64, device="cuda")
out = torch.empty_like(x)
alg = 4.0 * r.n_cells + 16.0 * r.n_padded
res = {}
for v in range(4):
    ssb.spmv_step_device(r, ssb.Variant(v), x, out)  # warm (plan built)
    ms = min(ssb.spmv_step_device(r, ssb.Variant(v), x, out) for _ in range(a.reps))
    res[["tropical", "real", "boolean", "selmax"][v]] = {"ms": round(ms, 3), "gbs": round(alg / ms / 1e6, 1),
                                                          "frac": round(alg / ms / 1e6 / peak, 3)}
print(json.dumps({"config": f"kronecker S{a.scale} C=32 sigma=n", "cells": r.n_cells, "rows": r.n_padded,
                  "algorithmic_bytes": int(alg), "peak_gbs": peak, "per_semiring": res}))
