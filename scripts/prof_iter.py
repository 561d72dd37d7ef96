"""Run the first --iters BFS iterations of one root (S --scale) twice: the second
launch is the one to profile (ncu -k regex:bfs32 -s 1 -c 1)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--root", type=int, default=2564265)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--variant", type=int, default=3)
ap.add_argument("--L", type=int, default=128)
ap.add_argument("--graph", default="kronecker", choices=["kronecker", "er"])
ap.add_argument("--g500", type=int, default=-1, help="use the i-th bench.py Graph500 root instead of --root")
a = ap.parse_args()
g = (ssb.gen_erdos_renyi(1 << a.scale, 16 / ((1 << a.scale) - 1), 1) if a.graph == "er"
     else ssb.gen_kronecker(a.scale, 16, 1))
r = ssb.build_slimsell(g, 32, g.num_vertices())
del g
if a.g500 >= 0:
    from bench import graph500_roots
    a.root = graph500_roots(r.degrees(), a.g500 + 1, 1)[a.g500]
    print("root", a.root)
db = ssb.DeviceBfs(r)
o = ssb.BfsOptions(variant=ssb.Variant(a.variant), slimwork=True, slimchunk_len=a.L, max_iterations=a.iters)
for _ in range(2):
    k, ms, st, rc = db.run(a.root, o)
    print(f"iters={k} device_ms={ms:.3f} kernel_ms={db.last_timing()[0]:.3f} swept={db.columns_swept()}",
          [(s.iteration, round(s.elapsed_ns / 1e6, 3), s.columns_processed, s.frontier_size) for s in st])
balg = 4.0 * 32 * db.columns_swept() + 3.0 * len(st) * r.n_padded / 8.0 + 8.0 * r.n_padded
print(f"algorithmic_bytes_last_launch={int(balg)} (bench.py b_alg: 128 B per swept column + 3 bitmaps/iter + 8 B/row)")
