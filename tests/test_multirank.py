"""Multi-rank host logic on CPU (gloo, world_size 2): chunk-range sharding with
the per-iteration frontier all-gather reproduces the single-process reference
result bit for bit (dist, sel-max parents incl. the root encoding, counters).
The per-rank sweep here is a plain numpy restatement of the 1-bit iteration
(test helper); on B200s it is the device kernel."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_09913_b200.sharding import ShardedFrontierExchange, partition_chunks, root_shard

KINF = np.iinfo(np.int64).max


def test_partition_chunks_balanced():
    rng = np.random.default_rng(0)
    cl = np.sort(rng.integers(0, 300, 5000))[::-1].copy()
    for world in (1, 2, 3, 8):
        rs = partition_chunks(cl, 32, world)
        assert rs[0][0] == 0 and rs[-1][1] == cl.shape[0]
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        cells = [int((32 * cl[b:e] + 1).sum()) for b, e in rs]
        assert max(cells) <= (sum(cells) / world) * 1.05 + 32 * cl.max()
    assert root_shard(range(10), 1, 4) == [1, 5, 9]


def test_partition_segments_snake_and_balance():
    """Round-robin segments: the k·W cell-balanced pieces of
    partition_chunks dealt in snake order — every piece owned once, k per
    rank, each rank's share of the head (hub) pieces and of the cells even."""
    from paper_2010_09913_b200.sharding import partition_segments
    rng = np.random.default_rng(1)
    cl = np.sort(rng.integers(0, 5000, 20000) ** 2 // 5000)[::-1].copy()
    for world, k in ((2, 4), (3, 2), (8, 4), (4, 1)):
        segs = partition_segments(cl, 32, world, k)
        pieces = partition_chunks(cl, 32, world * k)
        assert sorted(x for sg in segs for x in sg) == sorted(pieces)
        assert all(len(sg) == k for sg in segs)
        # snake: round 0 deals pieces 0..W-1 to ranks 0..W-1, round 1 back
        assert [sg[0] for sg in segs] == pieces[:world]
        if k > 1:
            assert [sg[1] for sg in segs] == pieces[world:2 * world][::-1]
        cells = [sum(int((32 * cl[b:e] + 1).sum()) for b, e in sg) for sg in segs]
        assert max(cells) <= (sum(cells) / world) * 1.05 + 2 * k * 32 * cl.max()
    with pytest.raises(ValueError):
        partition_segments(cl, 32, 2, 0)


def sweep_range(L, b, e, F, visited, k, root_code, level, parent, slimwork, Lseg):
    """One BFS iteration over chunks [b, e) in 1-bit form (C = 32)."""
    n = L.n
    newF = np.zeros(e - b, dtype=np.uint32)
    proc = skip = cols = subs = front = 0
    for i in range(b, e):
        real = (1 << min(32, n - 32 * i)) - 1
        if slimwork and visited[i] == real:
            skip += 1
            continue
        proc += 1
        cl = int(L.cl[i])
        cols += cl
        if Lseg > 0 and cl > 0:
            subs += (cl + Lseg - 1) // Lseg
        if cl == 0:
            continue
        grid = L.col[L.cs[i]: L.cs[i] + 32 * cl].reshape(cl, 32)
        cells = np.where(grid >= 0, grid, 0)
        bits = ((F[cells >> 5] >> (cells & 31)) & 1).astype(bool) & (grid >= 0)
        hit = bits.any(axis=0)
        mask = sum(1 << r for r in range(32) if hit[r])
        newly = mask & ~int(visited[i]) & real
        if newly:
            visited[i] |= newly
            newF[i - b] = newly
            front += bin(newly).count("1")
            for r in range(32):
                if (newly >> r) & 1:
                    row = 32 * i + r
                    level[row] = k
                    last = np.nonzero(bits[:, r])[0][-1]
                    parent[row] = root_code if k == 1 else int(grid[last, r])
    return newF, np.array([proc, skip, subs, cols, front], dtype=np.int64)


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Port
        port_ = Port()
        n, uv = port_.gen_kronecker(11, 16, 4)
        row, col = port_.to_csr(n, uv)
        L = port_.build_slimsell(n, row, col, 32, n)
        ranges = partition_chunks(L.cl, 32, world)
        b, e = ranges[rank]
        ex = ShardedFrontierExchange(ranges, L.n_chunks, dist)
        out = {}
        for root, slimwork, Lseg in ((3, True, 8), (int(L.perm[0]), False, 0), (700, True, 0)):
            root_pos = int(L.inv_perm[root])
            root_code = root  # sel-max compat encoding
            visited = np.zeros(L.n_chunks, dtype=np.uint32)
            F = np.zeros(L.n_chunks, dtype=np.uint32)
            visited[root_pos >> 5] |= np.uint32(1 << (root_pos & 31))
            F[root_pos >> 5] |= np.uint32(1 << (root_pos & 31))
            level = np.full(L.n_padded, -1, dtype=np.int64)
            parent = np.full(L.n_padded, -1, dtype=np.int64)
            level[root_pos], parent[root_pos] = 0, root_code
            stats = []
            k = 0
            while True:
                k += 1
                newF, st = sweep_range(L, b, e, F, visited, k, root_code, level, parent, slimwork, Lseg)
                res = ex.exchange(rank, newF)
                # replicated state: everyone ORs the gathered frontier into visited
                visited |= res.frontier
                F = res.frontier
                stats.append(st)
                if not res.any_new:
                    break
            tot = np.stack(stats)
            import torch
            t = torch.from_numpy(tot.copy())
            dist.all_reduce(t)
            lv = torch.from_numpy(np.where(level >= 0, level, KINF))
            pr = torch.from_numpy(parent.copy())
            gl = [torch.zeros_like(lv) for _ in range(world)]
            gp = [torch.zeros_like(pr) for _ in range(world)]
            dist.all_gather(gl, lv)
            dist.all_gather(gp, pr)
            lvl = np.full(L.n_padded, KINF, dtype=np.int64)
            par = np.full(L.n_padded, -1, dtype=np.int64)
            for r, (rb, re) in enumerate(ranges):
                lvl[32 * rb: 32 * re] = gl[r].numpy()[32 * rb: 32 * re]
                par[32 * rb: 32 * re] = gp[r].numpy()[32 * rb: 32 * re]
            lvl[root_pos], par[root_pos] = 0, root_code
            d = np.empty(n, dtype=np.int64)
            p = np.full(n, -1, dtype=np.int64)
            d[L.perm] = lvl[:n]
            reached = lvl[:n] != KINF
            p[L.perm[reached]] = L.perm[par[:n][reached]]
            ref = port_.bfs_spmv(L, root, 3, slimwork, Lseg)
            rows = [[int(r[c]) for c in (2, 3, 4, 5, 6)] for r in ref.stats]
            out[(root, slimwork, Lseg)] = (bool(np.array_equal(d, ref.dist)), bool(np.array_equal(p, ref.parent)),
                                           t.numpy().tolist() == rows, k == ref.iterations)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_chunk_sharded_bfs_world2_matches_reference():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for key, (d_ok, p_ok, st_ok, it_ok) in out.items():
        assert d_ok and p_ok and st_ok and it_ok, key


def test_bench_spawner_runs_n_ranks(tmp_path, capfd):
    """`bench.py --gpus N` outside torchrun re-launches the command as N ranks
    under torch.distributed.run (127.0.0.1); here with a gloo stand-in script
    that all-reduces and lets rank 0 print one line."""
    import json
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    script = tmp_path / "rank.py"
    script.write_text(
        "import json, os, sys, torch, torch.distributed as dist\n"
        "dist.init_process_group('gloo')\n"
        "t = torch.tensor([int(os.environ['RANK']) + 1])\n"
        "dist.all_reduce(t)\n"
        "if dist.get_rank() == 0:\n"
        "    print(json.dumps({'world': dist.get_world_size(), 'sum': int(t.item()), 'argv': sys.argv[1:]}))\n"
        "dist.destroy_process_group()\n")
    rc = bench.spawn_ranks(2, script=str(script), argv=["--gpus", "2", "--steps", "1"])
    assert rc == 0
    out = [ln for ln in capfd.readouterr().out.splitlines() if ln.startswith("{")]
    assert len(out) == 1
    d = json.loads(out[0])
    assert d == {"world": 2, "sum": 3, "argv": ["--gpus", "2", "--steps", "1"]}


def test_p2p_attach_failure_is_collective(tmp_path, capfd):
    """The fused exchange's window mapping is collective: when one rank cannot
    map its peers' windows, EVERY rank raises P2PUnavailable (bench.py then
    falls back to the NCCL exchange) instead of the others hanging in the
    barrier. Gloo ranks with a stand-in shard whose rank-1 attach fails."""
    import json
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "rank.py"
    script.write_text(
        "import json, os, sys\n"
        f"sys.path.insert(0, {root!r})\n"
        "import torch.distributed as dist\n"
        "from paper_2010_09913_b200.sharding import P2PShard, P2PUnavailable\n"
        "dist.init_process_group('gloo')\n"
        "class Fake:\n"
        "    def window_handle(self):\n"
        "        return bytes([dist.get_rank()])\n"
        "    def attach(self, rank, world, handles):\n"
        "        assert handles == [bytes([r]) for r in range(world)]\n"
        "        if rank == 1:\n"
        "            raise RuntimeError('ipc refused')\n"
        "out = 'attached'\n"
        "try:\n"
        "    P2PShard.attach_dist(Fake())\n"
        "except P2PUnavailable as e:\n"
        "    out = str(e)\n"
        "outs = [None] * dist.get_world_size()\n"
        "dist.all_gather_object(outs, out)\n"
        "if dist.get_rank() == 0:\n"
        "    print(json.dumps(outs))\n"
        "dist.destroy_process_group()\n")
    rc = bench.spawn_ranks(2, script=str(script), argv=[])
    assert rc == 0
    out = [ln for ln in capfd.readouterr().out.splitlines() if ln.startswith("[")]
    assert json.loads(out[0]) == ["rank 1: ipc refused"] * 2


def test_bench_default_decomposition():
    """N = 1: the single-GPU engine; N > 1: fused peer exchange when every GPU
    pair maps each other's memory and the backend is NCCL, else the NCCL
    all-gather form."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    class FakeCuda:
        def __init__(self, n, peer):
            self.n, self.peer = n, peer

        def device_count(self):
            return self.n

        def can_device_access_peer(self, i, j):
            return self.peer

    class FakeTorch:
        def __init__(self, n, peer):
            self.cuda = FakeCuda(n, peer)

    assert bench.choose_shard(FakeTorch(1, True), 1)[0] == "roots"
    assert bench.choose_shard(FakeTorch(8, True), 8)[0] == "p2p"
    assert bench.choose_shard(FakeTorch(8, False), 8)[0] == "chunks"
    assert bench.choose_shard(FakeTorch(1, True), 2)[0] == "chunks"  # ranks sharing one GPU
    old = os.environ.get("SSB_BENCH_BACKEND")
    os.environ["SSB_BENCH_BACKEND"] = "gloo"
    try:
        assert bench.choose_shard(FakeTorch(8, True), 8)[0] == "chunks"
    finally:
        if old is None:
            del os.environ["SSB_BENCH_BACKEND"]
        else:
            os.environ["SSB_BENCH_BACKEND"] = old


def test_native_partition_equals_python_partition():
    """ssb_ctx_build's partition (C++, libslimsell_b200.so — host code, no
    device needed) deals exactly the segments sharding.partition_segments
    does, so a single-process context and a torch.distributed job shard a
    layout identically."""
    import ctypes as C

    from paper_2010_09913_b200 import _lib as L
    from paper_2010_09913_b200.sharding import partition_segments
    rng = np.random.default_rng(7)
    for nc in (1, 5, 1000, 77777):
        cl = (rng.integers(0, 3000, nc) ** 2 // 3000)[::-1].astype(np.int32).copy()
        for world, k in ((1, 1), (2, 4), (3, 2), (8, 4), (5, 3)):
            out = np.zeros(2 * world * k, np.int64)
            rc = L.lib().ssb_partition_segments(cl.ctypes.data_as(L.i32p), nc, 32, world, k,
                                                out.ctypes.data_as(L.i64p))
            assert rc == 0
            py = partition_segments(cl, 32, world, k)
            assert out.reshape(world, k, 2).tolist() == [[list(p) for p in sg] for sg in py], (nc, world, k)


def test_fingerprints_numpy_torch_partial_and_roots(port):
    """ph64 on the host (numpy) and on a torch device agree, partial sums over
    disjoint rows add up to the whole (how sharded runs compare with the
    reference), and graph500_roots follows the reference's pick_roots stream
    (the oracle's so_pick_roots) with degree-0 vertices rejected."""
    import torch

    from paper_2010_09913_b200.fingerprint import (graph500_roots, ph64_format, ph64_np,
                                                   ph64_partial_torch, ph64_torch)
    v = np.random.default_rng(2).integers(-(1 << 62), 1 << 62, 300001).astype(np.int64)
    v[::7] = np.iinfo(np.int64).max
    t = torch.from_numpy(v)
    assert ph64_np(v) == ph64_torch(t) == ph64_np(v, block=4096)
    m = torch.from_numpy(np.random.default_rng(3).random(v.shape[0]) < 0.4)
    assert ph64_format(ph64_partial_torch(t, m) + ph64_partial_torch(t, ~m)) == ph64_np(v)
    n = 5000
    deg = np.random.default_rng(4).integers(0, 3, n)
    want = [int(x) for x in port.pick_roots(n, n, 1) if deg[x] > 0][:40]
    assert graph500_roots(deg, 40, 1) == want


class _FakeShard:
    """A numpy stand-in for sharding.DeviceShard (the 1-bit sweep of
    sweep_range over chunks [b, e)) so run_sharded_bfs's host logic runs on
    CPU: lockstep iterations, the all-gather, the counter sums, the
    iteration cap."""

    def __init__(self, L, b, e):
        import types
        self.L, self.b, self.e = L, b, e
        self.r = types.SimpleNamespace(n=L.n)

    def begin(self, root, opts):
        L = self.L
        self.k = 0
        self.sw, self.Lseg = bool(opts.slimwork), int(opts.slimchunk_len)
        self.root_code = root
        rp = int(L.inv_perm[root])
        self.visited = np.zeros(L.n_chunks, dtype=np.uint32)
        self.F = np.zeros(L.n_chunks, dtype=np.uint32)
        self.visited[rp >> 5] |= np.uint32(1 << (rp & 31))
        self.F[rp >> 5] |= np.uint32(1 << (rp & 31))
        self.level = np.full(L.n_padded, -1, dtype=np.int64)
        self.parent = np.full(L.n_padded, -1, dtype=np.int64)
        self.level[rp], self.parent[rp] = 0, root
        self.rp = rp

    def step(self):
        import torch

        from paper_2010_09913_b200.api import IterStats
        self.k += 1
        newF, st = sweep_range(self.L, self.b, self.e, self.F, self.visited, self.k, self.root_code,
                               self.level, self.parent, self.sw, self.Lseg)
        s = IterStats(self.k, 0, *[int(x) for x in st])
        return s, torch.from_numpy(newF.view(np.int32).copy())

    def exchange(self, full, newly_total):
        words = full.numpy().view(np.uint32)
        self.visited |= words
        self.F = words.copy()

    def fetch(self, want_parents, dist, parent):
        L = self.L
        for pos in range(32 * self.b, min(32 * self.e, L.n)):
            o = int(L.perm[pos])
            if self.level[pos] >= 0:
                dist[o] = self.level[pos]
                if want_parents:
                    parent[o] = int(L.perm[self.parent[pos]])
        if want_parents and self.b <= self.rp >> 5 < self.e:
            parent[int(L.perm[self.rp])] = int(L.perm[self.root_code])


def test_run_sharded_bfs_host_logic_and_cap(port):
    """sharding.run_sharded_bfs over two shards in one process (LocalComm):
    dist, sel-max parents (the reference's root encoding) and every counter
    equal the oracle; opts.max_iterations caps the BFS with BfsCapError
    carrying the partial distances and no parents (bfs.cpp:86-90)."""
    from paper_2010_09913_b200.api import BfsCapError, BfsOptions, Variant
    from paper_2010_09913_b200.sharding import LocalComm, run_sharded_bfs
    n, uv = port.gen_kronecker(10, 16, 9)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    ranges = partition_chunks(L.cl, 32, 2)
    shards = [_FakeShard(L, b, e) for b, e in ranges]
    for root in (3, 500):
        o = BfsOptions(variant=Variant.selmax, slimwork=True, slimchunk_len=8)
        dist_, parent, per_iter = run_sharded_bfs(shards, LocalComm(), root, o)
        ref = port.bfs_spmv(L, root, 3, True, 8)
        assert np.array_equal(dist_, ref.dist)
        assert np.array_equal(parent, ref.parent)
        assert [[s.chunks_processed, s.chunks_skipped, s.subchunks_processed, s.columns_processed,
                 s.frontier_size] for s in per_iter] == [[int(r[c]) for c in (2, 3, 4, 5, 6)] for r in ref.stats]
    o = BfsOptions(variant=Variant.selmax, slimwork=True, slimchunk_len=8, max_iterations=2)
    with pytest.raises(BfsCapError) as ei:
        run_sharded_bfs(shards, LocalComm(), 3, o)
    capped = port.bfs_spmv(L, 3, 3, True, 8, max_iterations=2)
    assert ei.value.partial.iterations == 2 and len(ei.value.partial.parent) == 0
    assert np.array_equal(ei.value.partial.dist, capped.dist)
