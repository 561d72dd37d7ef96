"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != "ID"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0][:64]
    t = float(r[14].replace(",", "")) * (1e-6 if r[13] == "ns" else 1e-3 if r[13] == "us" else 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
bfs = {k: v for k, v in agg.items() if any(s in k for s in ("bfs32", "set_root", "unpermute", "dp_parent", "reached_degree", "summary_from"))}
other = {k: v for k, v in agg.items() if k not in bfs}
for title, d in (("BFS path (per-root kernels)", bfs), ("graph generation + SlimSell build (once, outside the timed region)", other)):
    tot = sum(v[1] for v in d.values())
    print(f"\n## {title}\n{'kernel':<66}{'launches':>9}{'total_ms':>11}{'share':>8}")
    for k, v in sorted(d.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:<66}{v[0]:>9}{v[1]:>11.3f}{100*v[1]/tot:>7.1f}%")
