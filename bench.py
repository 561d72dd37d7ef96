#!/usr/bin/env python
"""bench.py — SlimSell BFS-SpMV on B200: GTEPS on a Graph500 Kronecker graph.

Workload (BASELINE.json config 3): gen_kronecker(26, 16, seed 1) built into
SlimSell with C = 32, σ = n; sel-max semiring, SlimWork on, SlimChunk
L = --slimchunk; the Graph500 root set (the reference's pick_roots stream,
cli.cpp:114-134, rejecting degree-0 vertices). One "step" = one BFS from every
root of the batch (--roots, default 64).

  value  = Σ_roots m_cc / Σ_roots t  (GTEPS; t = device time of the BFS, CUDA
           events on the launching stream; m_cc = edges in the root's
           component; graph resident in HBM)
  e2e    = the same through the public C-ABI with HOST outputs (dist +
           parent, int64[n] each, into pinned buffers) — copies inside: the
           step's root list through ssb_bfs_spmv_batch (each root's fetch
           overlapped with the next root's BFS); e2e.single_call = one
           ssb_bfs_spmv call per root
  roofline: bfs32_kernel, algorithmic bytes B_alg = 4·C·Σ_k cols_k
           + 3·iters·n_padded/8 + 8·n_padded per launch
  cpu_baseline: the reference library itself (oracle/_ref, built from
           /root/reference sources) on this host, all cores, one root.

--impl reference runs the reference's OWN path on the host cores: its
gen_kronecker / gen_erdos_renyi, build_slimsell and bfs_spmv (oracle/_ref,
compiled from the unmodified sources); no libslimsell_b200.so is loaded.

Multi-GPU: `--gpus N` without WORLD_SIZE re-launches itself under
torch.distributed.run with N ranks (one per GPU). N > 1 defaults to
north_star's decomposition — chunk-range shards (round-robin segments) with the
frontier exchange fused into the BFS kernel over peer-mapped memory (--shard
p2p) — and falls back to the NCCL all-gather form (--shard chunks) when the
GPUs cannot map each other's memory or the backend is not NCCL. --shard roots
is root-parallel (every rank holds the whole graph).

Parity in the bench: every root of the step is validated on the device against
the reference's deterministic rules (Graph500 edge checks + bit-exact parents:
sel-max max-position rule with the root encoding, or the smallest-id rule), and
compared with the reference's own recorded outputs (tests/golden/golden_big.json,
ph64 of dist and parent + every IterStats counter) where it holds that root.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DATA = {"kronecker": "synthetic (device Kronecker generator, bit-identical to the reference gen_kronecker)",
        "er": "synthetic (Erdos-Renyi generator, bit-identical to the reference gen_erdos_renyi)"}
METRIC = "GTEPS (Graph500 BFS) Kronecker scale 26 at 1/2/4/8 B200; % HBM roofline"
FALLBACK_HBM = 6650.0


# ---------------------------------------------------------------------------
def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--slimchunk", type=int, default=2048)
    ap.add_argument("--chunk-height", type=int, default=32,
                    help="SlimSell C (32 = the warp-wide engine; BASELINE config 1 uses C=8, sigma=C)")
    ap.add_argument("--sigma", default="n", help="sorting scope: an integer, 'n' or 'C' (cli.cpp:156)")
    ap.add_argument("--variant", default="selmax", choices=["tropical", "real", "boolean", "selmax"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--graph", default="kronecker", choices=["kronecker", "er"],
                    help="er: BASELINE config 4, gen_erdos_renyi(2^scale, avg_degree/(n-1), seed)")
    ap.add_argument("--avg-degree", type=float, default=16.0)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-slimwork", action="store_true")
    ap.add_argument("--no-validate", action="store_true")
    ap.add_argument("--shard", default=None, choices=["roots", "chunks", "p2p"],
                    help="multi-GPU decomposition (default: p2p for N > 1 when the GPUs map each "
                         "other's memory, else chunks; single GPU at N = 1): independent roots per "
                         "rank, chunk-range shards with a per-iteration NCCL frontier all-gather, or "
                         "chunk-range shards with the exchange fused into the BFS kernel (p2p)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="N > 1: skip the secondary root-parallel figure")
    ap.add_argument("--segments", type=int, default=4,
                    help="--shard p2p: chunk segments per rank, dealt round-robin (snake order)")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="--shard p2p at N=1: run this many ranks as one cooperative launch on "
                         "the single GPU (measures the fused exchange's overhead)")
    return ap.parse_args()


from paper_2010_09913_b200.fingerprint import graph500_roots, ph64_torch  # noqa: E402  (loads no .so)

GOLDEN_BIG = os.path.join(ROOT, "tests", "golden", "golden_big.json")
L2_BYTES = 126 << 20
L2_NOTE: dict = {}  # set by main() for layouts small enough to sit in L2
ROOT_RULE = "pick_roots stream (cli.cpp:114-134) rejecting degree 0"


def golden_entry(a):
    """The reference's recorded outputs for this workload's graph, if any
    (tests/golden/golden_big.json, written by tests/golden/make_golden_big.py
    from the unmodified reference): (entry, {(root, variant, slimwork, L): case})."""
    key = None
    if a.seed == 1 and a.graph == "kronecker" and a.edgefactor == 16:
        key = f"kron{a.scale}"
    elif a.seed == 1 and a.graph == "er" and a.avg_degree == 16.0:
        key = f"er{a.scale}"
    try:
        with open(GOLDEN_BIG) as f:
            e = json.load(f).get(key)
    except Exception:
        e = None
    if not e:
        return None, {}
    return e, {(c["root"], c["variant"], c["slimwork"], c["L"]): c for c in e.get("cases", [])}


def config_of(a, slimwork, n_roots, parallelism, **extra):
    """The workload description both arms print (same keys, same values)."""
    gdesc = (f"erdos-renyi n=2^{a.scale} avg degree {a.avg_degree:g} seed {a.seed}" if a.graph == "er"
             else f"kronecker scale {a.scale} ef {a.edgefactor} seed {a.seed}")
    cfg = {"workload": (f"{gdesc}, SlimSell C={a.chunk_height} sigma={a.sigma}, "
                        f"{a.variant}, "
                        f"slimwork={'on' if slimwork else 'off'}, slimchunk L={a.slimchunk}, "
                        f"{n_roots} Graph500 roots/step"),
           "graph": a.graph, "scale": a.scale, "edgefactor": a.edgefactor, "C": a.chunk_height, "sigma": a.sigma,
           "semiring": a.variant, "slimwork": slimwork, "slimchunk_len": a.slimchunk,
           "roots_per_step": n_roots, "root_rule": ROOT_RULE, "parallelism": parallelism,
           "l2": L2_NOTE.get("note", "inputs larger than L2 (col >> 126 MB); no flush needed")}
    cfg.update(extra)
    return cfg


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def profiled_traffic(a):
    """dram bytes per bfs32 launch from the committed ncu capture OF THIS
    WORKLOAD (graph, scale, semiring), or (None, None) when none exists."""
    p = os.path.join(ROOT, "profiles", "ncu_bfs32_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except Exception:
        return None, None
    for e in d.get("entries", []):
        m = e.get("match", {})
        if (m.get("graph"), m.get("scale"), m.get("variant")) == (a.graph, a.scale, a.variant):
            return e.get("dram_bytes_per_launch"), (
                f"{e.get('workload')}; algorithmic bytes of that launch "
                f"{e.get('algorithmic_bytes_same_launch')}; {e.get('source')}")
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def b_alg(stats, C: int, n_padded: int, swept=None) -> float:
    """Algorithmic HBM bytes of one BFS: 4·C bytes per column
    the sweeps needed — `swept` (ssb_bfs_columns_swept: early-exit sweeps stop
    a unit once all its rows are decided) or, without it, Σ columns_processed —
    plus three n/8 bitmaps per iteration and the level + parent rows."""
    cols = swept if swept is not None else sum(s.columns_processed for s in stats)
    return 4.0 * C * cols + 3.0 * len(stats) * n_padded / 8.0 + 8.0 * n_padded


RED_DEV = "cuda"  # device of the small reduction tensors (cpu under gloo)


def init_dist(torch, ssb, world, local):
    """One process per GPU (NCCL). SSB_BENCH_BACKEND=gloo runs the multi-rank
    control flow where ranks share a GPU (functional check only)."""
    global RED_DEV
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    ssb.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("SSB_BENCH_BACKEND", "nccl")
        if dist.is_initialized():  # re-entered (the p2p -> NCCL fallback): keep the group
            if backend != "nccl":
                RED_DEV = "cpu"
            return dev
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
            RED_DEV = "cpu"
    return dev


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
def build_graph(ssb, a, log):
    t0 = time.time()
    if a.graph == "er":
        n = 1 << a.scale
        g = ssb.gen_erdos_renyi(n, a.avg_degree / (n - 1), a.seed)
    else:
        g = ssb.gen_kronecker(a.scale, a.edgefactor, a.seed)
    t1 = time.time()
    n = g.num_vertices()
    sigma = n if a.sigma == "n" else (a.chunk_height if a.sigma == "C" else int(a.sigma))
    r = ssb.build_slimsell(g, a.chunk_height, sigma)
    t2 = time.time()
    m = g.num_edges()
    log(f"graph S{a.scale}: n={r.n} m={m} cells={r.n_cells} gen {t1 - t0:.2f}s build {t2 - t1:.2f}s")
    return g, r, m, t1 - t0, t2 - t1


def reference_repr(ssb, r, log):
    """Materialise the device-built layout as the reference's SlimSellRepr
    (bit-identical to build_slimsell — tests/test_gpu_parity.py pins the
    fingerprints up to S22), so the reference's stock bfs_spmv can run on it
    without 8 + 5 minutes of single-threaded generation and build."""
    import ctypes as C

    from oracle import Reference
    from paper_2010_09913_b200 import _lib as L

    t0 = time.time()
    col32 = r.col32()
    cs = np.empty(r.n_chunks, np.int64)
    cl = np.empty(r.n_chunks, np.int64)
    perm = np.empty(r.n, np.int64)
    inv = np.empty(r.n, np.int64)
    p = lambda x: x.ctypes.data_as(L.i64p)  # noqa: E731
    rc = L.lib().ssb_graph_export(r._h, None, p(cs), p(cl), p(perm), p(inv))
    assert rc == 0
    ref = Reference()
    rr = ref.repr_from_arrays(r.n, r.C, r.sigma, r.nonzeros, col32, cs, cl, perm, inv)
    del col32
    log(f"reference repr materialised in {time.time() - t0:.1f}s")
    return ref, rr


def cpu_reference_run(ref, rr, root, variant, slimwork, L, cores):
    t0 = time.time()
    out = ref.bfs_spmv(rr, root, variant, slimwork=slimwork, slimchunk_len=L, schedule=1, workers=cores,
                       want_parents=True)
    wall = time.time() - t0
    t = float(out.stats[:, 1].sum()) * 1e-9  # Σ IterStats.elapsed_ns (cli.cpp:46-50)
    return out, t, wall


def m_cc_of(dist: np.ndarray, deg: np.ndarray) -> int:
    return int(deg[dist != np.iinfo(np.int64).max].sum() // 2)


def validate_roots(ssb, torch, a, g, r, db, opts, roots, variant_id, pin_d, pin_p):
    """Bit-exact parity of every root, without the host oracle:
    * ssb_validate_bfs_exact — Graph500 edge checks + every parent equal to the
      reference's deterministic value (sel-max: perm of the max neighbour
      position one level up, root encoding at levels 0-1, bfs.cpp:94-101 /
      SURVEY.md App. A.3; tropical / real / boolean: the smallest-id neighbour
      one level up, dp_transform semiring.cpp:159-187). Edge checks + exact
      parents fix dist and parent uniquely.
    * the reference's own outputs where tests/golden/golden_big.json holds the
      root: ph64(dist), ph64(parent) and every IterStats counter."""
    t0 = time.time()
    gold, cases = golden_entry(a)
    compat = variant_id == 3  # the bench runs the reference's sel-max encoding
    exact = "selmax" if variant_id == 3 else "min"
    bad, first, g_cmp, g_eq, g_first = 0, None, 0, 0, None
    for root in roots:
        k, _, stats, _ = db.run(root, opts)
        dd, pp = db.fetch(True, pin_d, pin_p)  # parents: sel-max decode, else dp_transform
        rep = ssb.validate_bfs(g, root, dd, pp, selmax_compat=compat, exact=exact, layout=r)
        if rep is not None:
            bad += 1
            first = first or f"root {root}: {rep}"
        c = cases.get((root, variant_id, not a.no_slimwork, a.slimchunk))
        if c is not None:
            g_cmp += 1
            got = {"dist_ph": ph64_torch(torch.from_numpy(dd).cuda()),
                   "parent_ph": ph64_torch(torch.from_numpy(pp).cuda()) if c["parent_ph"] else None,
                   "stats": [[x.iteration, x.chunks_processed, x.chunks_skipped, x.subchunks_processed,
                              x.columns_processed, x.frontier_size] for x in stats]}
            diff = [key for key in ("dist_ph", "parent_ph", "stats") if got[key] != c[key]]
            if diff:
                g_first = g_first or f"root {root}: {diff} differ"
            else:
                g_eq += 1
    # the device queue BFS (independent of the SlimSell path) for the first root
    t = ssb.bfs_traditional(g, roots[0])
    db.run(roots[0], opts)
    dd, _ = db.fetch(False, pin_d, pin_p)
    return {"roots": len(roots), "roots_bit_exact": len(roots) - bad, "roots_failed": bad,
            "first_failure": first,
            "checks": "ssb_validate_bfs_exact: Graph500 edge checks (cli.cpp:73-112 + Graph500) and every "
                      "parent equal to the reference's deterministic rule (" +
                      ("sel-max max-position, root encoding at levels 0-1, bfs.cpp:94-101" if exact == "selmax"
                       else "smallest-id neighbour one level up, semiring.cpp:159-187") + ")",
            "reference_golden": {"roots_compared": g_cmp, "roots_equal": g_eq, "first_difference": g_first,
                                 "what": "ph64(dist), ph64(parent), every IterStats counter vs the unmodified "
                                         "reference's bfs_spmv (tests/golden/golden_big.json)"},
            "dist_equal_queue_bfs_first_root": bool(np.array_equal(dd, t.dist)),
            "seconds": round(time.time() - t0, 2)}


# ---------------------------------------------------------------------------
def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n: int, script: str | None = None, argv: list[str] | None = None) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1; rank 0
    prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script or os.path.abspath(__file__),
           *(sys.argv[1:] if argv is None else argv)]
    return subprocess.run(cmd).returncode


def peer_access_ok(torch, world: int) -> tuple[bool, str]:
    """Every pair of the first `world` GPUs can map each other's memory (the
    fused exchange's peer stores), and the collective backend is NCCL."""
    if os.environ.get("SSB_BENCH_BACKEND", "nccl") != "nccl":
        return False, "backend is not NCCL"
    if torch.cuda.device_count() < world:
        return False, f"{torch.cuda.device_count()} visible GPU(s) for {world} ranks"
    for i in range(world):
        for j in range(world):
            if i != j and not torch.cuda.can_device_access_peer(i, j):
                return False, f"GPU {i} cannot access GPU {j}"
    return True, "peer access between every pair"


def choose_shard(torch, world: int) -> tuple[str, str]:
    """Default decomposition: one GPU -> the single-GPU engine; N > 1 ->
    north_star's chunk-range shards, fused peer exchange when every pair of
    GPUs maps each other's memory, else the NCCL all-gather form."""
    if world <= 1:
        return "roots", "single GPU"
    ok, why = peer_access_ok(torch, world)
    return ("p2p" if ok else "chunks"), why


def main():
    a = args_()
    world, rank, local = dist_env()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a.gpus))
    log = (lambda *x: print("[bench]", *x, file=sys.stderr, flush=True)) if rank == 0 else (lambda *x: None)
    variant_id = {"tropical": 0, "real": 1, "boolean": 2, "selmax": 3}[a.variant]
    slimwork = not a.no_slimwork
    cores = os.cpu_count() or 1

    if a.impl == "reference":
        return main_reference(a, world, rank, local, log, variant_id, slimwork, cores)
    shard = a.shard
    if shard is None:
        import torch
        shard, why = choose_shard(torch, world)
        log(f"N={world}: --shard {shard} ({why})")
    if shard != "roots" and a.chunk_height != 32:
        raise SystemExit("the sharded BFS needs the C = 32 layout")
    if shard == "chunks":
        return main_chunks(a, world, rank, local, log, variant_id, slimwork)
    if shard == "p2p":
        why = None
        try:
            return main_p2p(a, world, rank, local, log, variant_id, slimwork)
        except Exception as e:  # every rank raises it together (sharding.P2PShard.attach_dist)
            if type(e).__name__ != "P2PUnavailable":
                raise
            why = str(e)
        log(f"fused peer exchange unavailable ({why}): --shard chunks")
        return main_chunks(a, world, rank, local, log, variant_id, slimwork)

    import torch

    import paper_2010_09913_b200 as ssb

    dev = init_dist(torch, ssb, world, local)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    g, r, m, t_gen, t_build = build_graph(ssb, a, log)
    deg = r.degrees()
    roots = graph500_roots(deg, a.roots, a.seed)
    mine = roots[rank::world]
    opts = ssb.BfsOptions(variant=ssb.Variant(variant_id), slimwork=slimwork, slimchunk_len=a.slimchunk)
    db = ssb.DeviceBfs(r)

    # warm-up (also computes m_cc per root once; the graph is static)
    mcc = {}
    for w in range(a.warmup):
        for root in mine:
            db.run(root, opts)
            if root not in mcc:
                mcc[root] = db.edges_traversed()
    for root in mine:
        if root not in mcc:
            db.run(root, opts)
            mcc[root] = db.edges_traversed()

    # ---- timed region: device time of K steps -------------------------------
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    step_ms, kern = [], []
    launches = 0
    per_root_ms = {}
    balg_total, kernel_ms_total, n_bfs = 0.0, 0.0, 0
    first_stats = None
    t_wall0 = time.time()
    # layouts that fit L2 (config 1's S16) get it flushed before every BFS
    flush = None
    if 4 * r.n_cells < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")
        L2_NOTE["note"] = (f"col = {4 * r.n_cells / 1e6:.1f} MB fits L2: a {2 * L2_BYTES >> 20} MB buffer is "
                           "written before every timed BFS (outside its CUDA-event interval)")
    for s in range(a.steps):
        tot = 0.0
        for root in mine:
            if flush is not None:
                flush.fill_(s)
                torch.cuda.synchronize()
            k, ms, stats, rc = db.run(root, opts)
            assert rc == 0, "BFS hit the iteration cap"
            kms, nl = db.last_timing()
            tot += ms
            launches += nl
            balg_total += b_alg(stats, r.C, r.n_padded, db.columns_swept())
            kernel_ms_total += kms
            n_bfs += 1
            per_root_ms.setdefault(root, []).append(ms)
            if first_stats is None:  # the step's first root (mine[0])
                first_stats = stats
        step_ms.append(tot)
    barrier()
    wall_s = time.time() - t_wall0
    clocks = sampler.stop()

    my_edges = sum(mcc[x] for x in mine)
    my_ms = float(np.mean(step_ms))
    tot_edges, max_ms = my_edges, my_ms
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(my_edges), my_ms], dtype=torch.float64, device=RED_DEV)
        e = t[:1].clone()
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        mx = t[1:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot_edges, max_ms = float(e.item()), float(mx.item())
    value = tot_edges / (max_ms * 1e-3) / 1e9

    # Graph500-style aggregates over roots (this rank)
    teps = [mcc[x] / (np.median(per_root_ms[x]) * 1e-3) / 1e9 for x in mine]
    hmean = len(teps) / sum(1.0 / t for t in teps)

    # ---- roofline of the dominant kernel ------------------------------------
    peak, peak_src = hbm_peak()
    achieved = balg_total / (kernel_ms_total * 1e-3) / 1e9
    traffic, traffic_src = profiled_traffic(a)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "bfs32_kernel" if r.C == 32 else "gen_chunk_kernel + gen_sweep_kernel (C != 32)",
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": round(balg_total / n_bfs),
                "kernel_ms_per_launch": round(kernel_ms_total / n_bfs, 4),
                "kernel_share_of_step": round(kernel_ms_total / max(sum(step_ms), 1e-9), 4)}
    if traffic_src:
        roofline["traffic_workload"] = traffic_src

    # ---- e2e: public C-ABI calls with host (pinned) outputs ------------------
    # The step's root list goes through ssb_bfs_spmv_batch (root i's result
    # crosses PCIe and is widened on the host while root i+1's BFS runs) into
    # two alternating pinned output pairs, as a double-buffering consumer
    # would; the per-root ssb_bfs_spmv loop is timed beside it.
    n = r.n
    pins = [(torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(),
             torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()) for _ in range(2)]
    pin_d, pin_p = pins[0]
    parents_out = variant_id == 3  # sel-max returns parents; the others need a CSR (dp_transform)
    # warm-up: both wire slots (device + pinned staging) allocated outside the timed region
    ssb.bfs_spmv_batch(r, mine[:2], opts, None, [pins[i % 2][0] for i in range(2)],
                       [pins[i % 2][1] for i in range(2)] if parents_out else None)
    barrier()
    t0 = time.time()
    e2e_edges = 0
    for s in range(a.e2e_steps):
        its = ssb.bfs_spmv_batch(r, mine, opts, None, [pins[i % 2][0] for i in range(len(mine))],
                                 [pins[i % 2][1] for i in range(len(mine))] if parents_out else None)
        e2e_edges += sum(mcc[x] for x in mine)
    barrier()
    e2e_s = time.time() - t0
    if a.e2e_steps:  # the e2e result must be a real BFS from the last root
        last = pins[(len(mine) - 1) % 2]
        assert int(last[0][mine[-1]]) == 0 and (not parents_out or int(last[1][mine[-1]]) >= 0)
    # the same through one ssb_bfs_spmv call per root (no overlap between roots)
    barrier()
    t1 = time.time()
    for root in mine:
        res = ssb.bfs_spmv(r, root, opts, None, pin_d, pin_p)
    barrier()
    single_s = time.time() - t1
    assert int(res.dist[mine[-1]]) == 0 and len(res.parent) == (n if parents_out else 0)
    e2e_tot, e2e_max = float(e2e_edges), e2e_s
    single_tot, single_max = float(sum(mcc[x] for x in mine)), single_s
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_tot, single_tot], dtype=torch.float64, device=RED_DEV)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        mx = torch.tensor([e2e_s, single_s], dtype=torch.float64, device=RED_DEV)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        e2e_tot, single_tot = float(t[0].item()), float(t[1].item())
        e2e_max, single_max = float(mx[0].item()), float(mx[1].item())
    wire = os.environ.get("SSB_WIRE", "1") != "0" and n >= 1 << 16  # fetch_rows' wire-format rule
    # bfs.cu wire_launch: sel-max dist + parents cross as ONE packed 32-bit word
    # (level << id_bits | parent id) when ids and levels fit (BFS depth here << 2^(32 - id_bits))
    id_bits = max(1, int(n - 1).bit_length())
    packed = (wire and parents_out and variant_id == 3 and id_bits <= 31
              and os.environ.get("SSB_WIRE_PACKED", "1") != "0")
    per_vertex = (4 if packed else (5 if parents_out else 1)) if wire else (16 if parents_out else 8)
    e2e = {"value": round(e2e_tot / e2e_max / 1e9, 3) if e2e_tot else None, "unit": "GTEPS",
           "h2d_bytes_per_step": 8 * len(roots),
           "d2h_bytes_per_step": per_vertex * n * len(roots),
           "note": "ssb_bfs_spmv_batch over the step's roots: roots in, dist" +
                   ("+parent" if parents_out else "") + " int64[n] per root out to pinned host memory" +
                   ((" (PCIe carries one packed 32-bit word per vertex, level << %d | parent id, "
                     "widened to int64 by host threads while the next root's BFS runs)" % id_bits) if packed else
                    (" (PCIe carries uint8 levels + int32 parents, widened to int64 by host threads "
                     "while the next root's BFS runs)" if wire else "")),
           "single_call": {"value": round(single_tot / single_max / 1e9, 3), "unit": "GTEPS",
                           "note": "one ssb_bfs_spmv call per root, same outputs"}}

    # ---- parity of every root of the step (device, untimed) -----------------
    validation = None
    if not a.no_validate:
        validation = validate_roots(ssb, torch, a, g, r, db, opts, mine, variant_id, pin_d, pin_p)
        log(f"validation: {validation}")

    # ---- CPU baseline: the reference library on this host, one root ---------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            ref, rr = reference_repr(ssb, r, log)
            root0 = mine[0]
            out, t, wall = cpu_reference_run(ref, rr, root0, variant_id, slimwork, a.slimchunk, cores)
            # parity of the sampled root while we have it
            db.run(root0, opts)
            dd, pp = db.fetch(True)
            same = bool(np.array_equal(dd, out.dist) and np.array_equal(pp, out.parent))
            cpu = {"value": round(mcc[root0] / t / 1e9, 5), "unit": "GTEPS", "cores": cores,
                   "kind": "reference", "cpu_model": lscpu_model(),
                   "sample": f"1 of {len(roots)} roots (root {root0}), full S{a.scale} graph; "
                             f"reference bfs_spmv, workers={cores}, dynamic_queue; t = Σ elapsed_ns "
                             f"{t:.2f}s (wall {wall:.2f}s)",
                   "bit_exact_vs_gpu": same}
            del rr
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GTEPS", "cores": cores, "kind": "reference",
                   "sample": f"unavailable: {type(ex).__name__}: {ex}"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(max_ms, 3),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": DATA[a.graph],
        "config": config_of(a, slimwork, len(roots), f"root-parallel x{world}" if world > 1 else "single GPU"),
        "graph_info": {"n": r.n, "m": m, "n_cells": r.n_cells, "col_gb_int32": round(4 * r.n_cells / 1e9, 2),
                       "iterations_first_root": len(first_stats), "first_root": mine[0]},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "validation": validation,
        "gpu_launches": int(launches),
        "graph500": {"harmonic_mean_gteps": round(hmean, 3), "median_gteps": round(float(np.median(teps)), 3),
                     "m_cc_first_root": mcc[mine[0]]},
        "timing": {"device_ms_steps": [round(x, 3) for x in step_ms], "host_wall_s": round(wall_s, 3),
                   "gen_s": round(t_gen, 3), "build_s": round(t_build, 3)},
        "per_iteration_first_root": [{"k": s.iteration, "ms": round(s.elapsed_ns / 1e6, 4),
                                      "cols": s.columns_processed, "frontier": s.frontier_size,
                                      "skipped": s.chunks_skipped} for s in first_stats],
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def sharded_parity(torch, dist_mod, world, a, roots, variant_id, slimwork, run_fetch, deg, n):
    """m_cc and reference parity of a sharded BFS without gathering vectors:
    each rank fetches its OWNED rows (other entries keep the -2 sentinel),
    sums their degrees and their ph64 terms; one all-reduce per root adds the
    ranks' partials (ph64 is a sum over positions)."""
    from paper_2010_09913_b200.fingerprint import ph64_format, ph64_partial_torch
    _, cases = golden_entry(a)
    mcc, g_cmp, g_eq = {}, 0, 0
    dd = np.empty(n, np.int64)
    pp = np.empty(n, np.int64)
    deg_t = torch.from_numpy(deg).cuda()
    for root in roots:
        dd.fill(-2)
        pp.fill(-2)
        run_fetch(root, dd, pp)
        td = torch.from_numpy(dd).cuda()
        mine = td != -2
        reached = mine & (td != np.iinfo(np.int64).max)
        deg_sum = int(deg_t[reached].sum().item())
        c = cases.get((root, variant_id, slimwork, a.slimchunk))
        parts = [deg_sum, 0, 0]
        if c is not None:
            parts[1] = ph64_partial_torch(td, mine)
            if variant_id == 3:
                tp = torch.from_numpy(pp).cuda()
                parts[2] = ph64_partial_torch(tp, tp != -2)
        t = torch.tensor(parts, dtype=torch.int64, device=RED_DEV)
        if world > 1:
            dist_mod.all_reduce(t)
        deg_tot, dph, pph = (int(x) for x in t.cpu().tolist())
        mcc[root] = deg_tot // 2
        if c is not None:
            g_cmp += 1
            g_eq += int(ph64_format(dph) == c["dist_ph"] and
                        (variant_id != 3 or ph64_format(pph) == c["parent_ph"]))
    return mcc, {"roots_compared": g_cmp, "roots_equal": g_eq,
                 "what": "ph64 of the assembled dist (and sel-max parent) vs the unmodified reference's "
                         "bfs_spmv (tests/golden/golden_big.json); partial sums over each rank's owned "
                         "rows, all-reduced"}


def sharded_e2e(torch, dist_mod, world, roots, run_fetch, mcc, variant_id, n):
    """e2e of a sharded BFS through the public calls with HOST outputs: every
    BFS of the step, then each rank's owned rows (int64 dist, + sel-max
    parents) into pinned host arrays (ssb_bfs_shard_fetch: the unpermute
    kernel writes them over PCIe); max over ranks."""
    pd = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    pp = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    run_fetch(roots[0], pd, pp)  # warm
    if world > 1:
        dist_mod.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for root in roots:
        run_fetch(root, pd, pp)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=RED_DEV)
    if world > 1:
        dist_mod.all_reduce(t, op=dist_mod.ReduceOp.MAX)
    per_row = 16 if variant_id == 3 else 8
    return {"value": round(sum(mcc[x] for x in roots) / float(t.item()) / 1e9, 3), "unit": "GTEPS",
            "h2d_bytes_per_step": 8 * len(roots), "d2h_bytes_per_step": per_row * n * len(roots),
            "note": "every root's BFS, then each rank's owned rows (int64 dist" +
                    (" + sel-max parent" if variant_id == 3 else "") + ") into pinned host arrays "
                    "(ssb_bfs_shard_fetch); host wall clock, max over ranks"}


def root_parallel_secondary(torch, dist_mod, ssb, a, world, rank, roots, opts, mcc):
    """The secondary figure at N > 1: every rank holds the WHOLE layout and
    runs roots[rank::N] with no collective (what root-parallel batches give on
    this box), timed like the primary line (device time, max over ranks)."""
    g = (ssb.gen_erdos_renyi(1 << a.scale, a.avg_degree / ((1 << a.scale) - 1), a.seed) if a.graph == "er"
         else ssb.gen_kronecker(a.scale, a.edgefactor, a.seed))
    r = ssb.build_slimsell(g, 32, g.num_vertices())
    del g
    db = ssb.DeviceBfs(r)
    mine = roots[rank::world]
    for root in mine:
        db.run(root, opts)
    if world > 1:
        dist_mod.barrier()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(a.steps):
        for root in mine:
            tot += db.run(root, opts)[1]
    t = torch.tensor([tot / a.steps], dtype=torch.float64, device=RED_DEV)
    if world > 1:
        dist_mod.all_reduce(t, op=dist_mod.ReduceOp.MAX)
    ms = float(t.item())
    del db, r
    return {"value": round(sum(mcc[x] for x in roots) / (ms * 1e-3) / 1e9, 3), "unit": "GTEPS",
            "ms_per_step": round(ms, 3),
            "what": "secondary: every rank holds the whole layout and runs roots[rank::N], no data-path collective"}


def shard_evidence(a, world, n_padded, iters_first, cells_rank, peak):
    """Exchange volume and its NVLink floor next to the HBM figures."""
    words = (n_padded + 31) // 32
    per_iter_rank_in = 4 * words * (world - 1) // max(world, 1)  # bytes each rank receives per iteration
    return {"frontier_words": words, "exchange_bytes_per_iteration_per_rank": per_iter_rank_in,
            "nvlink_gbs": 770.0, "nvlink_gbs_source": "measured peer copy per direction on this pool "
                                                      "(B200_PROFILING.md; nominal 900)",
            "nvlink_floor_us_per_iteration": round(per_iter_rank_in / 770e9 * 1e6, 2),
            "cells_per_rank": cells_rank, "iterations_first_root": iters_first,
            "hbm_peak_gbs": peak}


def main_chunks(a, world, rank, local, log, variant_id, slimwork):
    """Chunk-range sharding: every rank holds and sweeps its
    contiguous, cell-balanced chunk range (range build: its own cells only)
    plus the replicated 1-bit frontier; one all-gather of the owned frontier
    words per iteration. Under NCCL the iteration loop has no host round trip:
    the all-gather is enqueued on the shard's stream between the sweep and
    the exchange, |F| is counted on the device, and the host polls |F_{k-1}|
    while k is queued (sharding.run_sharded_bfs_async); counters are summed
    once per BFS. Under gloo (ranks sharing one GPU: a functional check) the
    words go through host memory and every step synchronises."""
    import torch

    import paper_2010_09913_b200 as ssb
    from paper_2010_09913_b200.sharding import DeviceShard, TorchComm, partition_chunks, run_sharded_bfs

    init_dist(torch, ssb, world, local)
    import torch.distributed as dist_mod

    def barrier():
        if world > 1:
            dist_mod.barrier()
        torch.cuda.synchronize()

    t0 = time.time()
    g = (ssb.gen_erdos_renyi(1 << a.scale, a.avg_degree / ((1 << a.scale) - 1), a.seed) if a.graph == "er"
         else ssb.gen_kronecker(a.scale, a.edgefactor, a.seed))
    t_gen = time.time() - t0
    n = g.num_vertices()
    meta = ssb.build_slimsell(g, 32, n, chunk_range=(0, 0))  # perm / cl / degrees, no cells
    deg = meta.degrees()
    roots = graph500_roots(deg, a.roots, a.seed)
    ranges = partition_chunks(meta.cl, 32, world)
    del meta
    t0 = time.time()
    r = ssb.build_slimsell(g, 32, n, chunk_range=ranges[rank])
    t_build = time.time() - t0
    log(f"graph S{a.scale}: n={n} m={g.num_edges()}; rank 0 holds chunks {ranges[0]} = {r.range_cells} of "
        f"{r.n_cells} cells; gen {t_gen:.2f}s build {t_build:.2f}s")
    del g
    shard = DeviceShard(r, *ranges[rank])

    class OneRank:  # N = 1: the same asynchronous loop, nothing to exchange
        device_async = True

        def allgather_frontier(self, owned_list):
            return owned_list[0]

        def allreduce_sum(self, arrays):
            return arrays[0]

    comm = TorchComm(ranges) if world > 1 else OneRank()
    mode = "async" if getattr(comm, "device_async", False) else "sync"
    opts = ssb.BfsOptions(variant=ssb.Variant(variant_id), slimwork=slimwork, slimchunk_len=a.slimchunk)
    launches = [0]

    def one(root):
        if mode == "async":
            _, _, per_iter = run_sharded_bfs([shard], comm, root, opts, fetch=False)
            ms = shard.last_ms  # CUDA events on the shard's stream around the whole BFS
        else:
            t = time.perf_counter()
            _, _, per_iter = run_sharded_bfs([shard], comm, root, opts, fetch=False)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t) * 1e3
        launches[0] += shard.launches()
        return ms, per_iter

    for _ in range(a.warmup):
        for root in roots:
            one(root)
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    step_ms = []
    launches[0] = 0
    first_iter = None
    swept = 0
    for s_ in range(a.steps):
        tot = 0.0
        for root in roots:
            ms, per_iter = one(root)
            tot += ms
            first_iter = first_iter or per_iter
            if s_ == 0:
                swept += ssb.DeviceBfs(r).columns_swept()
        step_ms.append(tot)
    barrier()
    clocks = sampler.stop()

    def run_fetch(root, dd, pp):
        run_sharded_bfs([shard], comm, root, opts, fetch=False)
        shard.fetch(variant_id == 3, dd, pp)

    mcc, golden = sharded_parity(torch, dist_mod, world, a, roots, variant_id, slimwork, run_fetch, deg, n)
    e2e = sharded_e2e(torch, dist_mod, world, roots, run_fetch, mcc, variant_id, n)
    secondary = None
    if world > 1 and not a.no_secondary:
        secondary = root_parallel_secondary(torch, dist_mod, ssb, a, world, rank, roots, opts, mcc)
    my_ms = float(np.mean(step_ms))
    t = torch.tensor([my_ms, swept], dtype=torch.float64, device=RED_DEV)
    per_rank_ms = [my_ms]
    if world > 1:
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist_mod.all_gather(allt, t)
        per_rank_ms = [float(x[0].item()) for x in allt]
        swept_all = [float(x[1].item()) for x in allt]
    else:
        swept_all = [float(swept)]
    max_ms = max(per_rank_ms)
    value = sum(mcc.values()) / (max_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    if world > 1:
        ct = torch.tensor([r.range_cells], dtype=torch.int64, device=RED_DEV)
        allc = [torch.zeros_like(ct) for _ in range(world)]
        dist_mod.all_gather(allc, ct)
        cells = [int(x.item()) for x in allc]
    else:
        cells = [r.range_cells]
    ev = shard_evidence(a, world, r.n_padded, len(first_iter), cells, peak)
    # HBM side: the busiest rank's swept col bytes per step over its time
    hbm_gbs = max(128.0 * sw for sw in swept_all) / (max_ms * 1e-3) / 1e9
    ev.update({"per_rank_ms_per_step": [round(x, 3) for x in per_rank_ms],
               "hbm_achieved_gbs_busiest_rank_col_stream": round(hbm_gbs, 1),
               "comm": (f"NCCL all_gather_into_tensor on the shard stream, {world} ranks" if world > 1 and
                        mode == "async" else ("gloo all_gather through host memory (functional)"
                                              if world > 1 else "single rank")),
               "stepping": mode})
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(max_ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": DATA[a.graph],
        "config": config_of(a, slimwork, len(roots), f"chunk-range shards x{world}, frontier all-gather"),
        "roofline": None, "cpu_baseline": None,
        "e2e": e2e,
        "clocks": clocks, "gpu_launches": int(launches[0]),
        "sharding": ev, "validation": {"reference_golden": golden}, "root_parallel": secondary,
        "timing": {"device_ms_steps": [round(x, 3) for x in step_ms], "gen_s": round(t_gen, 3),
                   "build_s": round(t_build, 3),
                   "clock": "CUDA events on the shard stream" if mode == "async" else
                            "host wall per BFS (gloo functional mode: every step synchronises)"},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist_mod.destroy_process_group()


def main_p2p(a, world, rank, local, log, variant_id, slimwork):
    """Chunk-range sharding with the frontier exchange FUSED into the BFS
    kernel (sharding.P2PShard): each rank's owned frontier words go straight
    into the peers' windows over NVLink and the ranks meet at an in-kernel
    counter barrier — one cooperative launch per BFS per rank. Needs one GPU
    per rank (ranks that wait on each other must not share a GPU); at N=1,
    --emulate-ranks W runs W ranks as one launch on the single GPU."""
    import torch

    import paper_2010_09913_b200 as ssb
    from paper_2010_09913_b200.sharding import P2PShard, partition_segments, run_p2p_group

    if world > 1 and torch.cuda.device_count() < world:
        raise SystemExit("--shard p2p needs one GPU per rank")
    dev = init_dist(torch, ssb, world, local)
    if world > 1 and os.environ.get("SSB_BENCH_BACKEND", "nccl") != "nccl":
        raise SystemExit("--shard p2p runs over NCCL ranks on separate GPUs")

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # every rank holds only its own chunks' cells: a
    # metadata-only build (empty range) gives cl for the partition, then each
    # rank builds its range — the memory that lets S28 span 8 GPUs
    t0 = time.time()
    g = (ssb.gen_erdos_renyi(1 << a.scale, a.avg_degree / ((1 << a.scale) - 1), a.seed) if a.graph == "er"
         else ssb.gen_kronecker(a.scale, a.edgefactor, a.seed))
    t_gen = time.time() - t0
    n = g.num_vertices()
    meta = ssb.build_slimsell(g, 32, n, chunk_range=(0, 0))
    deg = meta.degrees()
    roots = graph500_roots(deg, a.roots, a.seed)
    opts = ssb.BfsOptions(variant=ssb.Variant(variant_id), slimwork=slimwork, slimchunk_len=a.slimchunk)
    emu = max(1, a.emulate_ranks) if world == 1 else 1
    ranges = partition_segments(meta.cl, 32, emu if emu > 1 else world, max(1, a.segments))
    del meta
    t0 = time.time()
    if emu > 1:
        reprs = [ssb.build_slimsell(g, 32, n, segments=sg) for sg in ranges]
        r = reprs[0]
    else:
        r = ssb.build_slimsell(g, 32, n, segments=ranges[rank])
    t_build = time.time() - t0
    log(f"graph S{a.scale}: n={n} m={g.num_edges()}, cells of rank 0's range {r.range_cells} "
        f"of {r.n_cells}; gen {t_gen:.2f}s build {t_build:.2f}s")
    del g
    if emu > 1:

        def one(root, fetch=False):
            d, p, per_iter, ms = run_p2p_group(reprs, ranges, root, opts, fetch=fetch)
            return ms, d
    else:
        shard = P2PShard(r, ranges[rank])
        if world > 1:
            shard.attach_dist()
        else:
            shard.attach(0, 1, [shard.window_handle()])

        def one(root):
            k, ms, st = shard.run(root, opts)
            return ms, None

    for _ in range(a.warmup):
        for root in roots:
            one(root)
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    step_ms = []
    for s in range(a.steps):
        step_ms.append(sum(one(root)[0] for root in roots))
    barrier()
    clocks = sampler.stop()
    # m_cc and reference parity per root from each rank's owned rows
    import torch.distributed as dist_mod

    def run_fetch(root, dd, pp):
        if emu > 1:
            d, p, _, _ = run_p2p_group(reprs, ranges, root, opts, fetch=True)
            dd[:] = d
            if len(p):
                pp[:] = p
        else:
            one(root)
            shard.fetch(variant_id == 3, dd, pp)

    mcc, golden = sharded_parity(torch, dist_mod, world, a, roots, variant_id, slimwork, run_fetch, deg, n)
    e2e = sharded_e2e(torch, dist_mod, world, roots, run_fetch, mcc, variant_id, n)
    secondary = None
    if world > 1 and emu == 1 and not a.no_secondary:
        secondary = root_parallel_secondary(torch, dist_mod, ssb, a, world, rank, roots, opts, mcc)
    my_ms = float(np.mean(step_ms))
    per_rank_ms = [my_ms]
    cells = [x.range_cells for x in (reprs if emu > 1 else [r])]
    if world > 1:
        t = torch.tensor([my_ms, float(r.range_cells)], dtype=torch.float64, device=RED_DEV)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist_mod.all_gather(allt, t)
        per_rank_ms = [float(x[0].item()) for x in allt]
        cells = [int(x[1].item()) for x in allt]
    max_ms = max(per_rank_ms)
    value = sum(mcc.values()) / (max_ms * 1e-3) / 1e9
    peak, _ = hbm_peak()
    ev = shard_evidence(a, max(world, emu), r.n_padded, None, cells, peak)
    ev.update({"per_rank_ms_per_step": [round(x, 3) for x in per_rank_ms],
               "segments_per_rank": a.segments,
               "exchange": ("peer stores + atomicOr into every peer's IPC-mapped window, in-kernel counter "
                            "barrier (ld.acquire.sys); one cooperative launch per BFS per rank" if emu == 1 else
                            "ranks emulated in one cooperative launch; windows are plain device memory"),
               "peer_windows_mapped": (world - 1) if emu == 1 else 0})
    par = (f"chunk-range shards x{world} ({a.segments} round-robin segments each), fused in-kernel "
           f"frontier exchange" if emu == 1 else
           f"{emu} chunk-range shards ({a.segments} round-robin segments each) emulated in one launch on "
           f"1 GPU, fused in-kernel exchange")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(max_ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": DATA[a.graph],
        "config": config_of(a, slimwork, len(roots), par,
                            cells_per_rank_max=max(x.range_cells for x in (reprs if emu > 1 else [r])),
                            n_cells=r.n_cells),
        "roofline": None, "cpu_baseline": None,
        "e2e": e2e,
        "clocks": clocks, "gpu_launches": 2 * len(roots) * a.steps,
        "sharding": ev, "validation": {"reference_golden": golden}, "root_parallel": secondary,
        "timing": {"device_ms_steps": [round(x, 3) for x in step_ms], "gen_s": round(t_gen, 3),
                   "build_s": round(t_build, 3)},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist_mod.destroy_process_group()


def lscpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main_reference(a, world, rank, local, log, variant_id, slimwork, cores):
    """The reference's OWN path on this host (oracle/_ref: the unmodified
    reference compiled from its sources): gen_kronecker / gen_erdos_renyi
    (generator.cpp:15-89) -> build_slimsell (repr.cpp:84-131) -> bfs_spmv
    (bfs.cpp:234-246), workers = all host threads, dynamic queue. Nothing of
    this repo's device path is loaded in this process. Each timed step is one
    root of the 64-root Graph500 list (cycled) — a bounded sample of the step
    the GPU arm times. Under torchrun only rank 0 works."""
    if rank != 0:
        return
    from oracle import Reference

    budget_s = float(os.environ.get("SSB_REF_BUDGET_S", "1650"))  # the driver's step limit is 30 min
    T0 = time.time()
    R = Reference()
    t0 = time.time()
    if a.graph == "er":
        n_in = 1 << a.scale
        g = R.gen_erdos_renyi(n_in, a.avg_degree / (n_in - 1), a.seed)
    else:
        g = R.gen_kronecker(a.scale, a.edgefactor, a.seed)
    t_gen = time.time() - t0
    deg = g.degrees()
    roots = graph500_roots(deg, a.roots, a.seed)
    t0 = time.time()
    sigma = g.n if a.sigma == "n" else (a.chunk_height if a.sigma == "C" else int(a.sigma))
    rr = R.build_slimsell(g, a.chunk_height, sigma)
    if 4 * rr.n_cells < 2 * L2_BYTES:  # the same config note as the B200 arm
        L2_NOTE["note"] = (f"col = {4 * rr.n_cells / 1e6:.1f} MB fits L2: a {2 * L2_BYTES >> 20} MB buffer is "
                           "written before every timed BFS (outside its CUDA-event interval)")
    t_build = time.time() - t0
    log(f"reference graph S{a.scale}: n={g.n} m={g.m} cells={rr.n_cells}; gen_kronecker {t_gen:.1f}s "
        f"build_slimsell {t_build:.1f}s (single-threaded, the reference's own code)")
    gold, cases = golden_entry(a)
    t0 = time.time()
    fnv = {k: rr.fnv(k) for k in ("col", "cs", "cl", "perm")}
    fnv["edges"] = g.edges_fnv()
    layout_check = None
    if gold:
        gl = gold.get("layout", {})
        layout_check = all(fnv[k] == gl.get(f"{k}_fnv") for k in ("col", "cs", "cl", "perm")) and \
            fnv["edges"] == gold.get("edges_fnv")
    log(f"layout FNV {fnv} ({time.time() - t0:.1f}s); equal to tests/golden/golden_big.json: {layout_check}")

    times, edges, ran = [], [], []
    first_out = None
    for i in range(a.warmup + a.steps):
        root = roots[i % len(roots)]
        if i >= a.warmup and times and time.time() - T0 + 2 * np.mean(times) + 120 > budget_s:
            log(f"time budget: stopping after {len(times)} of {a.steps} timed roots")
            break
        out, t, wall = cpu_reference_run(R, rr, root, variant_id, slimwork, a.slimchunk, cores)
        log(f"reference root {root}: {t:.2f}s ({wall:.2f}s wall) iterations {out.iterations}")
        if first_out is None:
            first_out = (root, out)
        if i >= a.warmup:
            times.append(t)
            edges.append(m_cc_of(out.dist, deg))
            ran.append(root)
    value = sum(edges) / sum(times) / 1e9
    # the first root's output against the reference's recorded output
    bit_same = None
    root0, out0 = first_out  # root0 == roots[0]
    mcc0 = m_cc_of(out0.dist, deg)
    c = cases.get((root0, variant_id, slimwork, a.slimchunk))
    if c is not None:
        from paper_2010_09913_b200.fingerprint import ph64_np
        bit_same = ph64_np(out0.dist) == c["dist_ph"] and (
            c["parent_ph"] is None or ph64_np(out0.parent) == c["parent_ph"])
    del out0, first_out
    del rr
    # the queue BFS (bfs_traditional, bfs.cpp:248-291), one thread: the
    # Trad-BFS stand-in of BASELINE.md §3
    trad = None
    if time.time() - T0 + 200 < budget_s:
        _, _, it, ts = R.bfs_traditional_timed(g, roots[0], want=False)
        trad = {"value": round(mcc0 / ts / 1e9, 5) if ts > 0 else None,
                "unit": "GTEPS", "threads": 1, "root": roots[0], "seconds": round(ts, 3), "iterations": it}
        g.drop_csr()
    sample = (f"each timed step = 1 root of the {len(roots)}-root Graph500 list (cycled; {len(ran)} timed "
              f"after {a.warmup} warm-up roots), full S{a.scale} graph built by the reference itself "
              f"(gen {t_gen:.0f}s + build_slimsell {t_build:.0f}s, untimed); reference bfs_spmv "
              f"workers={cores} dynamic_queue; t = sum of IterStats.elapsed_ns (cli.cpp:46-50)")
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": "GTEPS", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(1e3 * float(np.mean(times)), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "impl": "reference",
        "config": config_of(a, slimwork, len(roots), "single GPU" if world == 1 else f"root-parallel x{world}"),
        "cpu_baseline": {"value": round(value, 5), "unit": "GTEPS", "cores": cores, "kind": "reference",
                         "cpu_model": lscpu_model(), "sample": sample,
                         "traditional_bfs_1_thread": trad},
        "e2e": {"value": round(value, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_path": {"gen_s": round(t_gen, 1), "build_slimsell_s": round(t_build, 1),
                           "layout_fnv": fnv, "layout_equals_recorded_reference": layout_check,
                           "first_root_equals_recorded_reference": bit_same,
                           "timed_roots": len(ran), "wall_s": round(time.time() - T0, 1),
                           "native_code": "oracle/_ref/libslimsell_ref.so only (no libslimsell_b200.so)"},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
