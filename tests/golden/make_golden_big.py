"""Generate tests/golden/golden_big.json — reference outputs at the BENCHMARK
configurations (BASELINE.json configs 2-4) from the UNMODIFIED reference.

Runs in the build container only (needs /root/reference compiled into
oracle/_ref by oracle/Makefile; S26 peaks at ≈52 GB of host RAM and ≈30 min
on 8 cores). The JSON is committed; the GPU tests and bench.py compare the
device's outputs with it, so nothing on the GPU box reads /root/reference.

    PYTHONPATH=. python tests/golden/make_golden_big.py --s22 --s26 --er26

Recorded per graph: edge-set and layout fingerprints (FNV-1a-64 over int64
little-endian arrays, as golden.json), the Graph500 root list, and per
(root, variant, SlimWork, L) the reference bfs_spmv's iterations, IterStats
rows ([iteration, chunks_processed, chunks_skipped, subchunks_processed,
columns_processed, frontier_size]) and dist / parent fingerprints — FNV and
the parallel ph64 (paper_2010_09913_b200/fingerprint.py). The queue BFS
(bfs_traditional, bfs.cpp:248-291) adds tropical/real/boolean parents
(== dp_transform's) for a few roots.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import Port, Reference, build  # noqa: E402
from paper_2010_09913_b200.fingerprint import graph500_roots, ph64_np  # noqa: E402

OUT = os.path.join(HERE, "golden_big.json")
WORKERS = os.cpu_count() or 8


def stats_rows(s):
    return [[int(r[0]), int(r[2]), int(r[3]), int(r[4]), int(r[5]), int(r[6])] for r in s]


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def graph_entry(P, R, g, kind, **kw):
    t0 = time.time()
    e = {"kind": kind, **kw, "n": g.n, "m": g.m, "edges_fnv": g.edges_fnv()}
    log(f"{kind} {kw}: n={g.n} m={g.m} edges hashed in {time.time() - t0:.1f}s")
    return e


def layout_entry(r):
    return {"C": r.C, "sigma": r.sigma, "n_cells": r.n_cells, "padding": r.padding,
            **{f"{k}_fnv": r.fnv(k) for k in ("col", "cs", "cl", "perm", "inv_perm")}}


def bfs_case(P, R, r, root, variant, sw, L, csr_graph=None):
    t0 = time.time()
    res = R.bfs_spmv(r, root, variant, slimwork=sw, slimchunk_len=L, workers=WORKERS, schedule=1,
                     csr_graph=csr_graph)
    assert res.status == 0
    c = {"root": root, "variant": variant, "slimwork": sw, "L": L, "iterations": res.iterations,
         "dist_fnv": P.fnv(res.dist), "dist_ph": ph64_np(res.dist),
         "parent_fnv": P.fnv(res.parent) if len(res.parent) else None,
         "parent_ph": ph64_np(res.parent) if len(res.parent) else None,
         "stats": stats_rows(res.stats), "ref_seconds": round(float(res.stats[:, 1].sum()) * 1e-9, 3),
         "m_cc": None}
    return c, res, time.time() - t0


def trad_case(P, R, g, root):
    d, p, it, sec = R.bfs_traditional_timed(g, root)
    return {"root": root, "iterations": it, "dist_fnv": P.fnv(d), "dist_ph": ph64_np(d),
            "parent_fnv": P.fnv(p), "parent_ph": ph64_np(p), "ref_seconds": round(sec, 3)}


def kron22(P, R):
    """Config 2: S22, all four semirings, 16 Graph500 roots, SlimWork on/off, L=2048."""
    t0 = time.time()
    g = R.gen_kronecker(22, 16, 1)
    e = graph_entry(P, R, g, "kronecker", scale=22, ef=16, seed=1)
    deg = g.degrees()
    roots = graph500_roots(deg, 16, 1)
    r = R.build_slimsell(g, 32, g.n)
    e["layout"] = layout_entry(r)
    e["roots"] = roots
    e["cases"] = []
    for root in roots:
        for v in range(4):
            for sw in (True, False):
                c, res, _ = bfs_case(P, R, r, root, v, sw, 2048, csr_graph=g)
                c["m_cc"] = int(deg[res.dist != np.iinfo(np.int64).max].sum() // 2)
                e["cases"].append(c)
    e["seconds"] = round(time.time() - t0, 1)
    log(f"S22 done in {e['seconds']}s")
    return e


def kron26(P, R, n_roots=64, trad_roots=4):
    """Config 3: S26, sel-max + SlimWork + SlimChunk L=2048, 64 Graph500 roots;
    plus root 30,478,752 (SURVEY.md §6.2 / §8(d)'s worked example)."""
    t0 = time.time()
    g = R.gen_kronecker(26, 16, 1)
    t_gen = time.time() - t0
    e = graph_entry(P, R, g, "kronecker", scale=26, ef=16, seed=1)
    e["ref_gen_seconds"] = round(t_gen, 1)
    deg = g.degrees()
    roots = graph500_roots(deg, n_roots, 1)
    t1 = time.time()
    r = R.build_slimsell(g, 32, g.n)
    e["ref_build_seconds"] = round(time.time() - t1, 1)
    log(f"S26 gen {t_gen:.0f}s build {e['ref_build_seconds']}s")
    e["layout"] = layout_entry(r)
    e["roots"] = roots
    e["cases"] = []
    for root in roots + [30478752]:
        c, res, wall = bfs_case(P, R, r, root, 3, True, 2048)
        c["m_cc"] = int(deg[res.dist != np.iinfo(np.int64).max].sum() // 2)
        e["cases"].append(c)
        log(f"S26 root {root}: {res.iterations} iterations, {c['ref_seconds']}s ({wall:.1f}s wall)")
    # tropical semiring (dist only without a CSR) for two roots: same dist
    for root in roots[:2]:
        c, res, _ = bfs_case(P, R, r, root, 0, True, 2048)
        e["cases"].append(c)
    del r
    # queue BFS: dist + the smallest-id parents that dp_transform returns for
    # tropical/real/boolean
    e["traditional"] = []
    for root in roots[:trad_roots]:
        e["traditional"].append(trad_case(P, R, g, root))
        log(f"S26 queue BFS root {root}: {e['traditional'][-1]['ref_seconds']}s")
    g.drop_csr()
    e["seconds"] = round(time.time() - t0, 1)
    return e


def er26(P, R, n_roots=16):
    """Config 4: Erdős–Rényi 2^26, avg degree 16, sel-max + SlimWork, L=2048."""
    t0 = time.time()
    n = 1 << 26
    g = R.gen_erdos_renyi(n, 16.0 / (n - 1), 1)
    e = graph_entry(P, R, g, "erdos_renyi", n_in=n, avg_degree=16, seed=1)
    e["ref_gen_seconds"] = round(time.time() - t0, 1)
    deg = g.degrees()
    roots = graph500_roots(deg, n_roots, 1)
    t1 = time.time()
    r = R.build_slimsell(g, 32, g.n)
    e["ref_build_seconds"] = round(time.time() - t1, 1)
    e["layout"] = layout_entry(r)
    e["roots"] = roots
    e["cases"] = []
    for root in roots:
        c, res, wall = bfs_case(P, R, r, root, 3, True, 2048)
        c["m_cc"] = int(deg[res.dist != np.iinfo(np.int64).max].sum() // 2)
        e["cases"].append(c)
        log(f"ER26 root {root}: {res.iterations} iterations, {c['ref_seconds']}s ({wall:.1f}s wall)")
    del r
    e["traditional"] = [trad_case(P, R, g, roots[0])]
    g.drop_csr()
    e["seconds"] = round(time.time() - t0, 1)
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s22", action="store_true")
    ap.add_argument("--s26", action="store_true")
    ap.add_argument("--er26", action="store_true")
    args = ap.parse_args()
    build()
    P, R = Port(), Reference()
    gold = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            gold = json.load(f)
    gold["generator"] = "tests/golden/make_golden_big.py (reference via oracle/_ref, %d workers)" % WORKERS
    for flag, key, fn in (("s22", "kron22", kron22), ("s26", "kron26", kron26), ("er26", "er26", er26)):
        if getattr(args, flag):
            gold[key] = fn(P, R)
            with open(OUT, "w") as f:  # checkpoint after every graph
                json.dump(gold, f, separators=(",", ":"))
            log(f"wrote {OUT} ({os.path.getsize(OUT) / 1e3:.0f} KB)")


if __name__ == "__main__":
    main()
