"""Generate tests/golden/golden.json from the UNMODIFIED reference library.

Runs in the build container only (it needs /root/reference, compiled into
oracle/_ref/libslimsell_ref.so by oracle/Makefile). The JSON it writes is
committed, so the GPU box never reads /root/reference.

    PYTHONPATH=. python tests/golden/make_golden.py [--big]

Fingerprints are FNV-1a-64 over little-endian int64 arrays.
Stats rows omit elapsed_ns: [iteration, chunks_processed, chunks_skipped,
subchunks_processed, columns_processed, frontier_size].
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import Port, Reference, build  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def stats_rows(s):
    return [[int(r[0]), int(r[2]), int(r[3]), int(r[4]), int(r[5]), int(r[6])] for r in s]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also S22 (≈1 min of reference CPU time)")
    args = ap.parse_args()
    build()
    P, R = Port(), Reference()
    gold = {"generator": "tests/golden/make_golden.py (reference via oracle/_ref)", "cases": []}
    t0 = time.time()

    # ---- 1. graph + layout fingerprints (cfg 1 graph) ------------------------
    graphs = {}
    for scale in (10, 16) + ((20, 22) if args.big else ()):
        g = R.gen_kronecker(scale, 16, 1)
        uv = g.edges()
        graphs[scale] = g
        entry = {"kind": "kronecker", "scale": scale, "ef": 16, "seed": 1, "n": g.n, "m": g.m,
                 "edges_fnv": P.fnv(uv), "layouts": []}
        for C_, sig in ((8, 8), (32, g.n), (8, 1)):
            r = R.build_slimsell(g, C_, sig)
            L = r.layout()
            entry["layouts"].append({"C": C_, "sigma_in": sig, "sigma": L.sigma, "n_cells": L.n_cells,
                                     "padding": L.padding, "col_fnv": P.fnv(L.col), "cs_fnv": P.fnv(L.cs),
                                     "cl_fnv": P.fnv(L.cl), "perm_fnv": P.fnv(L.perm)})
        gold.setdefault("graphs", []).append(entry)
        print(f"graph S{scale}: {time.time() - t0:.1f}s", flush=True)

    # ---- 2. config 1: S16, sel-max, C=8, sigma=C, pick_roots(random:16, 1) ---
    g16 = graphs[16]
    r16 = R.build_slimsell(g16, 8, 8)
    roots = [int(x) for x in P.pick_roots(g16.n, 16, 1)]
    gold["cfg1_roots"] = roots
    for root in roots:
        for sw, L_ in ((False, 0), (True, 4), (True, 0)):
            res = R.bfs_spmv(r16, root, 3, slimwork=sw, slimchunk_len=L_, workers=8, schedule=1)
            gold["cases"].append({"graph": "kron16", "C": 8, "sigma": 8, "root": root, "variant": 3,
                                  "slimwork": sw, "L": L_, "iterations": res.iterations,
                                  "dist_fnv": P.fnv(res.dist), "parent_fnv": P.fnv(res.parent),
                                  "stats": stats_rows(res.stats)})
    # all four semirings at C=32, sigma=n on the same graph (fast engine)
    r16b = R.build_slimsell(g16, 32, g16.n)
    for root in roots[:4]:
        for v in range(4):
            res = R.bfs_spmv(r16b, root, v, slimwork=True, slimchunk_len=64, workers=8, schedule=1,
                             csr_graph=g16)
            gold["cases"].append({"graph": "kron16", "C": 32, "sigma": g16.n, "root": root, "variant": v,
                                  "slimwork": True, "L": 64, "iterations": res.iterations,
                                  "dist_fnv": P.fnv(res.dist), "parent_fnv": P.fnv(res.parent),
                                  "stats": stats_rows(res.stats)})
    print(f"cfg1: {time.time() - t0:.1f}s", flush=True)

    # ---- 3. small full vectors (S10, every semiring) ---------------------------
    g10 = graphs[10]
    full = []
    for C_, sig in ((32, g10.n), (8, 1), (8, 8)):
        r = R.build_slimsell(g10, C_, sig)
        for root in (0, 5, 700):
            for v in range(4):
                res = R.bfs_spmv(r, root, v, slimwork=True, slimchunk_len=4, workers=2, csr_graph=g10)
                full.append({"C": C_, "sigma": sig, "root": root, "variant": v, "iterations": res.iterations,
                             "dist": [int(x) for x in res.dist], "parent": [int(x) for x in res.parent],
                             "stats": stats_rows(res.stats)})
    gold["kron10_full"] = full

    # ---- 4. kernel-level spmv_step on random int64 vectors (S10, C=8, σ=8) ---
    r = R.build_slimsell(g10, 8, 8)
    rng = np.random.default_rng(5)
    sp = []
    for v in range(4):
        if v == 0:
            x = rng.integers(0, 50, r.n_padded)
            x[rng.random(r.n_padded) < 0.3] = np.iinfo(np.int64).max
        elif v == 1:
            x = rng.integers(-100, 100, r.n_padded)
        elif v == 2:
            x = rng.integers(0, 2, r.n_padded)
        else:
            x = rng.integers(0, 1000, r.n_padded)
        out = R.spmv_step(r, v, x)
        sp.append({"variant": v, "x": [int(a) for a in x], "out_fnv": P.fnv(out)})
    gold["kron10_spmv_C8_s8"] = sp

    # ---- 5. larger graphs: S20 (and S22 with --big) --------------------------
    big = [(20, [0, 70048])] if args.big else []
    if args.big:
        big.append((22, [0]))
    for scale, rts in big:
        g = graphs[scale]
        r = R.build_slimsell(g, 32, g.n)
        for root in rts:
            for v in range(4):
                res = R.bfs_spmv(r, root, v, slimwork=True, slimchunk_len=128, workers=8, schedule=1,
                                 csr_graph=g)
                gold["cases"].append({"graph": f"kron{scale}", "C": 32, "sigma": g.n, "root": root,
                                      "variant": v, "slimwork": True, "L": 128, "iterations": res.iterations,
                                      "dist_fnv": P.fnv(res.dist), "parent_fnv": P.fnv(res.parent),
                                      "stats": stats_rows(res.stats)})
        print(f"S{scale}: {time.time() - t0:.1f}s", flush=True)

    # ---- 6. the reference's own selftest verdict (documents the quirk) -------
    rc, text = R.selftest()
    gold["ref_selftest"] = {"exit": rc, "fail_lines": [ln for ln in text.splitlines() if ln.startswith("FAIL")]}

    with open(OUT, "w") as f:
        json.dump(gold, f, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
