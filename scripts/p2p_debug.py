"""Debug the emulated fused multi-GPU BFS at scale: per-root timing of the
group launch for a few world sizes (run under `timeout`, SSB_TRACE=1 polls)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2010_09913_b200 as ssb
from bench import graph500_roots
from paper_2010_09913_b200.sharding import partition_chunks, run_p2p_group
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
worlds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,3,2").split(",")]
g = ssb.gen_kronecker(scale, 16, 1)
reprs = [ssb.build_slimsell(g, 32, g.num_vertices()) for _ in range(max(worlds))]
roots = graph500_roots(reprs[0].degrees(), 8, 1)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
ref = {}
for w in worlds:
    ranges = partition_chunks(reprs[0].cl, 32, w)
    print("world", w, "ranges", ranges, flush=True)
    for root in roots:
        t = time.time()
        d, p, st, ms = run_p2p_group(reprs[:w], ranges, root, o)
        same = ""
        if root in ref:
            same = f" same={np.array_equal(ref[root][0], d) and np.array_equal(ref[root][1], p)}"
        else:
            ref[root] = (d, p)
        print(f"  root {root}: {len(st)} iters device {ms:.2f} ms wall {time.time() - t:.2f} s{same}", flush=True)
