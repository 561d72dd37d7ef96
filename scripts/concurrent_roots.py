"""Experiment: two BFS of the Graph500 root list at once, each on half the SMs
(SSB_GRID CTAs, two graph handles, two host threads), against the sequential
full-grid engine. Checks every root's dist/parent fingerprint equal."""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_09913_b200 as ssb
from paper_2010_09913_b200.fingerprint import graph500_roots, ph64_np

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--graph", default="kron")
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--split", type=int, default=2)
a = ap.parse_args()
ssb.set_device(0)
if a.graph == "er":
    n = 1 << a.scale
    g = ssb.gen_erdos_renyi(n, 16.0 / (n - 1), 1)
else:
    g = ssb.gen_kronecker(a.scale, 16, 1)
n = g.num_vertices()
rs = [ssb.build_slimsell(g, 32, n) for _ in range(a.split)]
roots = graph500_roots(rs[0].degrees(), a.roots, 1)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
dbs = [ssb.DeviceBfs(r) for r in rs]

def check(db, root):
    dist, par = db.fetch(True)
    return ph64_np(dist) + ph64_np(par)

os.environ["SSB_GRID"] = "148"
ref = {}
for root in roots:
    dbs[0].run(root, o)
    ref[root] = check(dbs[0], root)
for rep in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev_ms = 0.0
    for root in roots:
        dev_ms += dbs[0].run(root, o)[1]
    torch.cuda.synchronize()
    seq = time.perf_counter() - t0
    print(f"S{a.scale} sequential full grid: wall {seq*1e3:.2f} ms, device sum {dev_ms:.2f} ms", flush=True)
for grid in (148 // a.split, 148 // a.split - 2):
    os.environ["SSB_GRID"] = str(grid)
    bad = []
    for rep in range(a.reps + 1):
        def work(i):
            for root in roots[i::a.split]:
                dbs[i].run(root, o)
                if rep == 0 and check(dbs[i], root) != ref[root]:
                    bad.append(root)
        ths = [threading.Thread(target=work, args=(i,)) for i in range(a.split)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        torch.cuda.synchronize()
        w = time.perf_counter() - t0
        if rep:
            print(f"S{a.scale} {a.split} concurrent x {grid} CTAs: wall {w*1e3:.2f} ms", flush=True)
    print("mismatching roots:", bad, flush=True)
