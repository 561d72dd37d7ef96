"""Where a BFS's device interval goes outside bfs32_kernel (SSB_GAPS=1 lines:
host prepare, t0 -> kernel start, kernel end -> stats copy done)."""
import os
import re
import subprocess
import sys

if os.environ.get("SSB_GAPS") != "1":
    env = dict(os.environ, SSB_GAPS="1")
    out = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    pre = [float(x) for x in re.findall(r"host prepare32 ([\d.]+) us", out.stderr)]
    bef = [float(x) for x in re.findall(r"before last launch ([\d.]+) us", out.stderr)]
    aft = [float(x) for x in re.findall(r"after it ([\d.]+) us", out.stderr)]
    dev = [float(x) for x in re.findall(r"device ([\d.]+) ms", out.stderr)]
    k = len(dev) // 2  # second half: warm
    med = lambda v: sorted(v[-k:])[k // 2] if v else None  # noqa: E731
    print(out.stdout.strip())
    print(f"median over {k} warm BFS: host prepare32 {med(pre)} us, t0->kernel {med(bef)} us, "
          f"kernel end->stats copy {med(aft)} us, device {med(dev)} ms")
    sys.exit(out.returncode)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_09913_b200 as ssb  # noqa: E402
from paper_2010_09913_b200.fingerprint import graph500_roots  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ssb.set_device(0)
g = ssb.gen_kronecker(scale, 16, 1)
r = ssb.build_slimsell(g, 32, g.num_vertices())
roots = graph500_roots(r.degrees(), 32, 1)
db = ssb.DeviceBfs(r)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
for rep in range(2):
    for root in roots:
        db.run(root, o)
print(f"S{scale}: kernel ms {db.last_timing()}")
