"""Attribute an .ncu-rep's SASS stall samples / instructions to kernel-body
source lines (outermost inline call site) of bfs32_kernel<sel>.
usage: ncu_regions.py REP LIB.so [sel=1] [N]"""
import collections, csv, io, re, subprocess, sys, tempfile, os

rep, lib = sys.argv[1], sys.argv[2]
sel = sys.argv[3] if len(sys.argv) > 3 else "1"
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 30
SRC = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2010_09913_b200", "csrc",
                        "bfs.cu")).read().splitlines()
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = os.path.join(tmp, "bfs.sm_100a.cubin")
sass = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
fn = f"bfs32_kernelILb{sel}ELi{os.environ.get('KS', '8')}EEEvNS0_6Args32E:"
addr_site = {}
on = False
chain = []
in_hdr = False
for line in sass.splitlines():
    if line.endswith(fn) and not line.startswith("."):
        on = True
        continue
    if not on:
        continue
    if line.startswith(".L_x") or line.startswith("\t.section") or line.startswith("//-----"):
        if line.startswith("//-----"):
            break
    m = re.match(r'\s*//## File ".*?", line (\d+)(.*)', line)
    if m:
        if not in_hdr:
            chain = [int(m.group(1))]
            in_hdr = True
        chain += [int(x) for x in re.findall(r'inlined at ".*?", line (\d+)', m.group(2))]
        continue
    in_hdr = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
    if m and chain:
        # skip the run_tasks lambda call (kernel body -> lambda) level
        c = list(chain)
        # skip the kernel -> bfs32_body and body -> run_tasks lambda levels
        while len(c) > 1 and ("run_tasks(" in SRC[c[-1] - 1] or "bfs32_body<" in SRC[c[-1] - 1]):
            c = c[:-1]
        addr_site[int(m.group(1), 16)] = (c[-1], c[-2] if len(c) > 1 else c[-1])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
# one section per profiled launch ("Kernel Name" row, header row, SASS rows): take section LAUNCH
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        secs.append(cur)
    elif cur is not None:
        cur.append(r)
sec = secs[int(os.environ.get("LAUNCH", "0"))]
h = sec[0]; data = [r for r in sec[1:] if r and r[0].startswith("0x")]
iA = h.index("Address"); iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
base = min(int(r[iA], 16) for r in data)
agg = collections.defaultdict(lambda: [0, 0])
agg2 = collections.defaultdict(lambda: [0, 0])
for r in data:
    off = int(r[iA], 16) - base
    site = addr_site.get(off, (-1, -1))
    s = int(r[iS]) if r[iS].isdigit() else 0
    e = int(r[iE]) if r[iE].isdigit() else 0
    agg[site[0]][0] += s; agg[site[0]][1] += e
    agg2[site][0] += s; agg2[site][1] += e
T = sum(v[0] for v in agg.values()); E = sum(v[1] for v in agg.values())
srcl = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2010_09913_b200", "csrc", "bfs.cu")).read().splitlines()
print(f"samples {T} instructions {E}; by kernel-body line:")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:ntop]:
    txt = srcl[k - 1].strip()[:80] if k > 0 else "?"
    print(f"{k:>5} {100*v[0]/T:5.1f}% samp {100*v[1]/E:5.1f}% inst  {txt}")
print("by (body line, next level):")
for k, v in sorted(agg2.items(), key=lambda kv: -kv[1][0])[:ntop]:
    txt = srcl[k[1] - 1].strip()[:70] if k[1] > 0 else "?"
    print(f"{k[0]:>5}/{k[1]:<5} {100*v[0]/T:5.1f}% samp {100*v[1]/E:5.1f}% inst  {txt}")
if os.environ.get("DEEP"):
    # innermost source line (any depth) inside take_cells / Probe
    print("by innermost line:")
    inner = collections.Counter()
    for a, (ch) in addr_site.items():
        pass
