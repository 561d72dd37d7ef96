"""Where a step's device time goes, per BFS iteration, averaged over the
Graph500 roots of bench.py (no profiler: the engine's own %globaltimer
per-iteration records)."""
import argparse, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
from paper_2010_09913_b200.fingerprint import graph500_roots
ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--graph", default="kronecker")
ap.add_argument("--variant", type=int, default=3)
ap.add_argument("--roots", type=int, default=64)
ap.add_argument("--L", type=int, default=2048)
a = ap.parse_args()
g = (ssb.gen_erdos_renyi(1 << a.scale, 16 / ((1 << a.scale) - 1), 1) if a.graph == "er"
     else ssb.gen_kronecker(a.scale, 16, 1))
r = ssb.build_slimsell(g, 32, g.num_vertices())
del g
roots = graph500_roots(r.degrees(), a.roots, 1)
db = ssb.DeviceBfs(r)
o = ssb.BfsOptions(variant=ssb.Variant(a.variant), slimwork=True, slimchunk_len=a.L)
for root in roots[:4]:
    db.run(root, o)
per_k, tot, kern = {}, 0.0, 0.0
for root in roots:
    k, ms, st, rc = db.run(root, o)
    tot += ms
    kern += db.last_timing()[0]
    for s in st:
        d = per_k.setdefault(s.iteration, [0, 0.0, 0, 0])
        d[0] += 1
        d[1] += s.elapsed_ns / 1e6
        d[2] += s.columns_processed
        d[3] += s.frontier_size
out = {"config": f"{a.graph} S{a.scale} variant {a.variant} L {a.L}", "roots": len(roots),
       "ms_per_bfs": round(tot / len(roots), 4), "kernel_ms_per_bfs": round(kern / len(roots), 4),
       "per_k": {k: {"roots": v[0], "ms_per_bfs": round(v[1] / len(roots), 4),
                     "mean_cols": int(v[2] / v[0]), "mean_front": int(v[3] / v[0])} for k, v in sorted(per_k.items())}}
print(json.dumps(out))
