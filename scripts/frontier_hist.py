"""Where the BFS frontier of each level lies in the permuted (degree-sorted)
order, and how well 256- / 32-vertex summaries would filter probes."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--root", type=int, default=2564265)
ap.add_argument("--graph", default="kronecker")
ap.add_argument("--P", type=int, default=1 << 20)
a = ap.parse_args()
g = (ssb.gen_erdos_renyi(1 << a.scale, 16 / ((1 << a.scale) - 1), 1) if a.graph == "er"
     else ssb.gen_kronecker(a.scale, 16, 1))
r = ssb.build_slimsell(g, 32, g.num_vertices())
del g
db = ssb.DeviceBfs(r)
db.run(a.root, ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048))
dist, _ = db.fetch(False)
inv = r.inv_perm
n = r.n
pos_level = np.full(n, -1, np.int64)
pos_level[inv] = np.where(dist == np.iinfo(np.int64).max, -1, dist)
deg = np.empty(n, np.int64)
ssb._lib.lib().ssb_graph_degrees(r._h, deg.ctypes.data_as(ssb._lib.i64p))
degp = np.empty(n, np.int64); degp[inv] = deg
print("n", n, "isolated", int((deg == 0).sum()))
for k in range(0, int(pos_level.max()) + 1):
    f = np.nonzero(pos_level == k)[0]
    if len(f) == 0:
        continue
    inP = (f < a.P).sum()
    tail = f[f >= a.P]
    b256 = np.unique(tail >> 8).size
    b32 = np.unique(tail >> 5).size
    nb256 = (n - a.P) >> 8
    nb32 = (n - a.P) >> 5
    # probe-weighted: fraction of adjacency cells (cells ~ degree) whose target lies in a set block
    w = degp  # cells pointing at vertex v = deg(v)
    set256 = np.zeros(nb256 + 1, bool); set256[(tail - a.P) >> 8] = True
    set32 = np.zeros(nb32 + 1, bool); set32[(tail - a.P) >> 5] = True
    tv = np.arange(a.P, n)
    cells_tail = w[a.P:].sum()
    c256 = w[a.P:][set256[(tv - a.P) >> 8]].sum()
    c32 = w[a.P:][set32[(tv - a.P) >> 5]].sum()
    print(f"level {k}: |F|={len(f)} in prefix {inP} ({100*inP/len(f):.1f}%), tail blocks set: "
          f"256 {b256}/{nb256} ({100*b256/nb256:.1f}%), 32 {b32}/{nb32} ({100*b32/nb32:.1f}%); "
          f"tail-cell share needing exact: 256 {100*c256/max(cells_tail,1):.1f}% 32 {100*c32/max(cells_tail,1):.1f}%; "
          f"tail cells / all cells {100*cells_tail/w.sum():.1f}%")
