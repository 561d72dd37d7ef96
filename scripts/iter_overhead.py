import sys, time
sys.path.insert(0, "/root/repo")
import paper_2010_09913_b200 as ssb
for n in (2000, 8000):
    g = ssb.gen_path(n)
    r = ssb.build_slimsell(g, 32, n)
    db = ssb.DeviceBfs(r)
    o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
    for _ in range(2):
        k, ms, st, rc = db.run(0, o)
    print(n, "iters", k, "device_ms", round(ms, 3), "per-iter us", round(1000 * ms / k, 2), db.last_timing())
