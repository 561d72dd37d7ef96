"""Breakdown of the e2e path (ssb_bfs_spmv with host outputs) at S26."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_09913_b200 as ssb
g = ssb.gen_kronecker(26, 16, 1); r = ssb.build_slimsell(g, 32, g.num_vertices()); del g
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
n = r.n
pd = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
pp = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
db = ssb.DeviceBfs(r)
for it in range(3):
    t0 = time.perf_counter(); k, ms, st, rc = db.run(2564265, o); t1 = time.perf_counter()
    db.fetch(True, pd, pp); t2 = time.perf_counter()
    res = ssb.bfs_spmv(r, 2564265, o, None, pd, pp); t3 = time.perf_counter()
    print(f"run {1e3*(t1-t0):.2f} ms (device {ms:.2f})  fetch {1e3*(t2-t1):.2f} ms  bfs_spmv {1e3*(t3-t2):.2f} ms")
a = torch.empty(n, dtype=torch.int64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3): torch.from_numpy(pd).copy_(a, non_blocking=True)
torch.cuda.synchronize(); print(f"torch D2H pinned {3*8*n/(time.perf_counter()-t0)/1e9:.1f} GB/s")
