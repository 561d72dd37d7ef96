"""Instructions executed / stall samples of an .ncu-rep by INNERMOST source
line of bfs.cu (inlined helpers included). usage: ncu_lines.py REP LIB.so [sel] [N]"""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep, lib = sys.argv[1], sys.argv[2]
sel = sys.argv[3] if len(sys.argv) > 3 else "1"
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 40
SRC = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2010_09913_b200", "csrc",
                        "bfs.cu")).read().splitlines()
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, "bfs.sm_100a.cubin")], capture_output=True,
                      text=True).stdout
# bfs32_kernel<sel, S, hashed> (HASH=0/1: the hashed-summary instantiation)
fn = f"bfs32_kernelILb{sel}ELi{os.environ.get('KS', '8')}ELb{os.environ.get('HASH', '1')}EEEvNS0_6Args32E:"
site, on, cur, hdr = {}, False, None, False
for line in sass.splitlines():
    if line.endswith(fn) and not line.startswith("."):
        on = True
        continue
    if not on:
        continue
    if line.startswith("//-----"):
        break
    m = re.match(r'\s*//## File "(.*?)", line (\d+)', line)
    if m:
        if not hdr:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            hdr = True
        continue
    hdr = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(\S+)", line)
    if m and cur:
        site[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
secs, sec = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        sec = []
        secs.append(sec)
    elif sec is not None:
        sec.append(r)
sec = secs[int(os.environ.get("LAUNCH", "0"))]
h = sec[0]
data = [r for r in sec[1:] if r and r[0].startswith("0x")]
iA, iS, iE = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
iO = h.index("Source") if "Source" in h else None
base = min(int(r[iA], 16) for r in data)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in data:
    s = site.get(int(r[iA], 16) - base, ("?", -1))
    a = agg[s]
    a[0] += int(r[iS]) if r[iS].isdigit() else 0
    e = int(r[iE]) if r[iE].isdigit() else 0
    a[1] += e
    if iO is not None and e:
        a[2][r[iO].split()[0] if r[iO].split() else "?"] += e
T = sum(v[0] for v in agg.values()) or 1
E = sum(v[1] for v in agg.values()) or 1
print(f"samples {T} instructions {E}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:ntop]:
    txt = SRC[k[1] - 1].strip()[:70] if k[0] == "bfs.cu" and k[1] > 0 else str(k)
    ops = " ".join(f"{o}:{n * 100 // v[1]}" for o, n in v[2].most_common(4)) if v[1] else ""
    print(f"{k[1]:>5} {100 * v[1] / E:5.1f}% inst {100 * v[0] / T:5.1f}% samp  {txt:<70} [{ops}]")
