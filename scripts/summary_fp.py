"""How often a tail cell's frontier-summary bit is set (so the sweep pays an
exact L2 lookup) under the block summary (one bit per 256 consecutive
positions, the kernel's S = 8 summary) and under a hashed summary of the same
size (one multiplicative-hash bit per tail frontier vertex), for iterations 3
and 4 of S26 sel-max roots. Counts only cells of rows still unvisited at the
iteration (the ones the early-exit sweep probes). Analysis tool, not timed."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb
from paper_2010_09913_b200.fingerprint import graph500_roots

scale = int(os.environ.get("SCALE", "26"))
g = ssb.gen_kronecker(scale, 16, 1)
r = ssb.build_slimsell(g, 32, g.num_vertices())
del g
n = r.n
roots = graph500_roots(r.degrees(), 64, 1)
perm = torch.from_numpy(r.perm).cuda()          # perm[pos] = original id
inv = torch.from_numpy(r.inv_perm).cuda()
assert int((inv[perm[:1000]] - torch.arange(1000, device='cuda')).abs().max()) == 0
col = torch.from_numpy(r.col32()).cuda()
cl = torch.from_numpy(r.cl).cuda()
nch = cl.numel()
chunk_of = torch.repeat_interleave(torch.arange(nch, device='cuda', dtype=torch.int32), (cl * 32))
NW = (r.n_padded + 31) // 32
budget = 160 * 1024 // 4 - 4
SW = (((NW + 7) >> 3) + 31) // 32
SW = (SW + 3) // 4 * 4
PW = (budget - SW) // 8 * 8
P = PW * 32
HB = SW * 32
hb_log = HB.bit_length() - 1
print(f"S{scale}: P={P} summary bits={HB} cells={col.numel()}", flush=True)
db = ssb.DeviceBfs(r)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
KINF = np.iinfo(np.int64).max
step = 1 << 28
for root in roots[: int(os.environ.get("ROOTS", "16"))]:
    k_, ms, st, rc = db.run(int(root), o)
    dist, _ = db.fetch(False)
    d = torch.from_numpy(np.where(dist == KINF, 1 << 30, dist).astype(np.int32)).cuda()
    lvl = d[perm]  # by position
    out = {"root": int(root), "k3_ms": round(st[2].elapsed_ns / 1e6, 3), "F2": int(st[1].frontier_size)}
    for k in (3, 4):
        F = (lvl == k - 1)
        ftail = torch.nonzero(F[P:]).flatten() + P
        blk = torch.zeros(n // 256 + 1, dtype=torch.bool, device='cuda'); blk[ftail >> 8] = True
        hsh = torch.zeros(HB, dtype=torch.bool, device='cuda')
        hsh[((ftail.to(torch.int64) * 0x9E3779B1) & 0xffffffff) >> (32 - hb_log)] = True
        tot = tr = bs = hs = 0
        for b in range(0, col.numel(), step):
            c = col[b:b + step]
            rows = chunk_of[b:b + step].to(torch.int64) * 32 + (torch.arange(b, b + c.numel(), device='cuda') & 31)
            m = (c >= P) & (lvl[rows.clamp(max=n - 1)] >= k) & (rows < n)
            cc = c[m].to(torch.int64)
            tot += cc.numel()
            tr += int(F[cc].sum())
            bs += int(blk[cc >> 8].sum())
            hs += int(hsh[((cc * 0x9E3779B1) & 0xffffffff) >> (32 - hb_log)].sum())
        out[f"k{k}"] = {"F_tail": int(ftail.numel()), "open_tail_cells": tot, "true": tr,
                        "block_set": bs, "hash_set": hs,
                        "block_frac": round(bs / max(tot, 1), 4), "hash_frac": round(hs / max(tot, 1), 4)}
    print(json.dumps(out), flush=True)
