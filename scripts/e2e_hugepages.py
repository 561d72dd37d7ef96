"""e2e of ssb_bfs_spmv_batch into output buffers backed by 4 KB pages
(torch pin_memory) vs transparent huge pages (mmap + MADV_HUGEPAGE, then
cudaHostRegister): the host widening is bound by host-memory stores."""
import ctypes, mmap, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_09913_b200 as ssb
from paper_2010_09913_b200.fingerprint import graph500_roots
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), flush=True)
g = ssb.gen_kronecker(26, 16, 1); r = ssb.build_slimsell(g, 32, g.num_vertices()); del g
roots = graph500_roots(r.degrees(), 32, 1)
o = ssb.BfsOptions(variant=ssb.Variant.selmax, slimwork=True, slimchunk_len=2048)
n = r.n
db = ssb.DeviceBfs(r)
mcc = 0
for x in roots:
    db.run(x, o); mcc += db.edges_traversed()
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None

def thp_array(nbytes, register=True):
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.int64)
    a[:] = 0  # fault in (huge pages when THP allows)
    if register:
        ptr = a.ctypes.data
        rc = torch.cuda.cudart().cudaHostRegister(ptr, nbytes, 0)
        assert rc == 0 or int(rc) == 0, rc
    return a, m

def run(pins, label):
    ssb.bfs_spmv_batch(r, roots[:2], o, None, [pins[i % 2][0] for i in range(2)], [pins[i % 2][1] for i in range(2)])
    best = 1e9
    for _ in range(2):
        t0 = time.perf_counter()
        ssb.bfs_spmv_batch(r, roots, o, None, [pins[i % 2][0] for i in range(len(roots))],
                           [pins[i % 2][1] for i in range(len(roots))])
        best = min(best, time.perf_counter() - t0)
    print(f"{label}: e2e {mcc / best / 1e9:.2f} GTEPS ({1e3 * best / len(roots):.2f} ms/root)", flush=True)

torch_pins = [(torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(), torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()) for _ in range(2)]
run(torch_pins, "torch pin_memory (4 KB pages)")
keep = []
thp = []
for _ in range(2):
    a, m1 = thp_array(8 * n); b, m2 = thp_array(8 * n); keep += [m1, m2]; thp.append((a, b))
print("AnonHugePages:", [l for l in open("/proc/meminfo") if "AnonHugePages" in l][0].strip(), flush=True)
run(thp, "THP + cudaHostRegister")
thp_np = []
for _ in range(2):
    a, m1 = thp_array(8 * n, register=False); b, m2 = thp_array(8 * n, register=False); keep += [m1, m2]; thp_np.append((a, b))
run(thp_np, "THP pageable (staged)")
run(torch_pins, "torch pin_memory again")
