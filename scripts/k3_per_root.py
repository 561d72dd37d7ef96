"""Per-root iteration-3 cost at S26 (sel-max): |F_2|, the mode the kernel
picks (dense / direct thresholds as bfs.cu's prepare32), ms, columns."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
from paper_2010_09913_b200.fingerprint import graph500_roots
g = ssb.gen_kronecker(26, 16, 1); r = ssb.build_slimsell(g, 32, g.num_vertices()); del g
roots = graph500_roots(r.degrees(), 64, 1)
db = ssb.DeviceBfs(r)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
dense_thr, direct_thr = r.n // 8192, 262144
rows = []
for x in roots:
    k, ms, st, rc = db.run(x, o)
    f2 = st[1].frontier_size
    mode = "direct" if f2 > direct_thr else ("dense" if f2 > dense_thr else "sparse")
    rows.append((st[2].elapsed_ns / 1e6, f2, mode, st[2].columns_processed, st[2].frontier_size, st[3].elapsed_ns / 1e6, x))
rows.sort()
for r_ in rows:
    print("k3 %.3f ms  F2 %8d %-6s cols %9d found %9d | k4 %.3f ms  root %d" % r_)
