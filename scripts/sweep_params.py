"""Parameter sweep on one S26 graph: GTEPS over a root batch for each
(slimchunk L, SSB_WARP_COLS, ...) combination (env knobs read per BFS)."""
import argparse, itertools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2010_09913_b200 as ssb
from bench import graph500_roots
ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--roots", type=int, default=16)
ap.add_argument("--L", default="128,256,512")
ap.add_argument("--env", action="append", default=[], help="NAME=v1,v2,...")
ap.add_argument("--graph", default="kronecker", choices=["kronecker", "er"])
ap.add_argument("--variant", type=int, default=3)
ap.add_argument("--reps", type=int, default=1, help="repeat the whole combination list (interleaved A/B)")
a = ap.parse_args()
g = (ssb.gen_erdos_renyi(1 << a.scale, 16 / ((1 << a.scale) - 1), 1) if a.graph == "er"
     else ssb.gen_kronecker(a.scale, 16, 1))
r = ssb.build_slimsell(g, 32, g.num_vertices())
del g
roots = graph500_roots(r.degrees(), a.roots, 1)
db = ssb.DeviceBfs(r)
envs = [(e.split("=")[0], e.split("=")[1].split(",")) for e in a.env]
combos = list(itertools.product([int(x) for x in a.L.split(",")], *[v for _, v in envs])) * a.reps
mcc = {}
for combo in combos:
    L = combo[0]
    for (name, _), val in zip(envs, combo[1:]):
        os.environ[name] = val
    o = ssb.BfsOptions(variant=ssb.Variant(a.variant), slimwork=True, slimchunk_len=L)
    db.run(roots[0], o)  # warm (plan build)
    tot_ms, tot_e, kms = 0.0, 0, 0.0
    for root in roots:
        k, ms, st, rc = db.run(root, o)
        if root not in mcc:
            mcc[root] = db.edges_traversed()
        tot_ms += ms
        kms += db.last_timing()[0]
        tot_e += mcc[root]
    print(f"L={L} " + " ".join(f"{n}={v}" for (n, _), v in zip(envs, combo[1:])) +
          f"  GTEPS={tot_e / tot_ms / 1e6:.2f}  kernel_ms/bfs={kms / len(roots):.3f}", flush=True)
