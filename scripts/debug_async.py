import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
from oracle import Port
from paper_2010_09913_b200.sharding import DeviceShard, partition_chunks
os.environ["SSB_SMEM_KB"] = "4"
port = Port()
n, uv = port.gen_kronecker(15, 16, 2)
g = ssb.Graph.from_pairs(uv, n)
row, col = port.to_csr(n, uv)
L = port.build_slimsell(n, row, col, 32, n)
r = ssb.build_slimsell(g, 32, n)
sh = DeviceShard(r, 0, r.n_chunks)
for root in (0, 5, 2000):
    for v, sw, Lc in ((3, True, 64), (0, True, 0), (3, False, 0), (2, True, 2048)):
        o = ssb.BfsOptions(variant=ssb.Variant(v), slimwork=sw, slimchunk_len=Lc)
        sh.begin_async(root, o)
        fr = []
        with torch.cuda.stream(sh.stream()):
            for k in range(1, 12):
                owned = sh.step_async()
                sh.exchange_async(owned)
                fr.append(sh.front(k))
        loc, ms = sh.finish(11)
        b = port.bfs_spmv(L, root, v, sw, Lc)
        print(root, v, sw, Lc, "front", fr, "local", [s.frontier_size for s in loc], "oracle",
              [int(x) for x in b.stats[:, 6]])
