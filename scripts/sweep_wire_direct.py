"""e2e of ssb_bfs_spmv_batch (S26 sel-max, Graph500 roots, pinned int64
outputs) for several shares of direct (DMA int64) fetch chunks
(SSB_WIRE_DIRECT — an experiment that was reverted; only 0 exists now), each checked equal to the wire-only output."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_09913_b200 as ssb
from paper_2010_09913_b200.fingerprint import graph500_roots, ph64_torch
g = ssb.gen_kronecker(26, 16, 1); r = ssb.build_slimsell(g, 32, g.num_vertices()); del g
roots = graph500_roots(r.degrees(), int(sys.argv[1]) if len(sys.argv) > 1 else 16, 1)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
n = r.n
pins = [(torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(), torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()) for _ in range(2)]
db = ssb.DeviceBfs(r)
mcc = {}
for x in roots:
    db.run(x, o); mcc[x] = db.edges_traversed()
ref = None
for pct in [int(x) for x in os.environ.get("PCTS", "0").split(",")]:
    os.environ["SSB_WIRE_DIRECT"] = str(pct)
    ssb.bfs_spmv_batch(r, roots[:2], o, None, [pins[i % 2][0] for i in range(2)], [pins[i % 2][1] for i in range(2)])
    t0 = time.perf_counter()
    ssb.bfs_spmv_batch(r, roots, o, None, [pins[i % 2][0] for i in range(len(roots))], [pins[i % 2][1] for i in range(len(roots))])
    dt = time.perf_counter() - t0
    last = pins[(len(roots) - 1) % 2]
    h = (ph64_torch(torch.from_numpy(last[0]).cuda()), ph64_torch(torch.from_numpy(last[1]).cuda()))
    ref = ref or h
    print(f"pct {pct:3d}: e2e {sum(mcc.values()) / dt / 1e9:.2f} GTEPS ({1e3 * dt / len(roots):.2f} ms/root) same={h == ref}", flush=True)
