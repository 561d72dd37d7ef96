"""Summarise an ab_env.sh / ab_run.sh log: ms per BFS and per iteration."""
import json, re, sys
for line in open(sys.argv[1]):
    m = re.match(r'(lib|env)=(\[.*?\]|\S+) rep=(\d) (.*)', line.strip())
    if not m:
        continue
    try:
        d = json.loads(m.group(4))
    except ValueError:
        print(line.strip()[:200]); continue
    print(m.group(2).split('/')[-1], m.group(3), d['config'], d['ms_per_bfs'], d['kernel_ms_per_bfs'],
          ' '.join(f"{k}:{v['ms_per_bfs']}" for k, v in d['per_k'].items()))
