"""GPU suite: the sm_100a path through the C-ABI against the oracle and the
reference's golden vectors. Bit-exact everywhere (integer path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINF = np.iinfo(np.int64).max
STAT_KEYS = ("iteration", "chunks_processed", "chunks_skipped", "subchunks_processed",
             "columns_processed", "frontier_size")


def dev_rows(res):
    return [[getattr(s, k) for k in STAT_KEYS] for s in res.per_iter]


def port_rows(stats):
    return [[int(r[c]) for c in (0, 2, 3, 4, 5, 6)] for r in stats]


def opts(ssb, v, slimwork=False, L=0, compat=True, max_it=0):
    return ssb.BfsOptions(variant=ssb.Variant(v), slimwork=slimwork, slimchunk_len=L,
                          selmax_compat=compat, max_iterations=max_it)


# ---- graph input + builder --------------------------------------------------

@pytest.mark.parametrize("scale", [10, 16, 20, 22])
def test_device_kronecker_and_builder_match_reference(ssb, port, golden, scale):
    e = next(g for g in golden["graphs"] if g["scale"] == scale)
    g = ssb.gen_kronecker(scale, 16, 1)
    assert (g.num_vertices(), g.num_edges()) == (e["n"], e["m"])
    assert port.fnv(g.edges()) == e["edges_fnv"]
    for lay in e["layouts"]:
        r = ssb.build_slimsell(g, lay["C"], lay["sigma_in"])
        assert (r.sigma, r.n_cells, r.padding) == (lay["sigma"], lay["n_cells"], lay["padding"])
        assert port.fnv(r.col) == lay["col_fnv"]
        assert port.fnv(r.cs) == lay["cs_fnv"]
        assert port.fnv(r.cl) == lay["cl_fnv"]
        assert port.fnv(r.perm) == lay["perm_fnv"]
        assert np.array_equal(r.inv_perm[r.perm], np.arange(r.n))


def test_from_pairs_and_csr_match_oracle(ssb, port):
    rng = np.random.default_rng(1)
    for n in (1, 2, 7, 300):
        pairs = rng.integers(0, n, size=(5 * n + 3, 2))
        pairs = np.concatenate([pairs, pairs[:5], np.stack([np.arange(n)] * 2, 1)])  # dups + loops
        g = ssb.Graph.from_pairs(pairs, n)
        nn, uv = port.from_pairs(pairs, n)
        assert g.num_vertices() == nn and np.array_equal(g.edges(), uv)
        csr = ssb.to_csr(g)
        row, col = port.to_csr(nn, uv)
        assert np.array_equal(csr.row, row) and np.array_equal(csr.col, col)
    g = ssb.Graph.from_pairs(np.array([[0, 5], [2, 3]]))  # inferred n
    assert g.num_vertices() == 6 and g.edges().tolist() == [[0, 5], [2, 3]]
    assert ssb.Graph.from_pairs(np.zeros((0, 2), np.int64), 0).num_vertices() == 0
    with pytest.raises(ssb.OutOfRange):
        ssb.Graph.from_pairs(np.array([[0, 9]]), 5)
    with pytest.raises(ssb.OutOfRange):
        ssb.Graph.from_pairs(np.array([[-1, 2]]))


def small_graphs(port):
    """The reference selftest's graph list (cli.cpp:360-382), seed 7."""
    out = [("path7", *port.gen_path(7)), ("clique5", *port.gen_clique(5)), ("star9", *port.gen_star(9))]
    idx, seed = 0, 7
    for n in (16, 33, 64):
        for p in (0.05, 0.15, 0.4):
            out.append((f"er{n}_{p}", *port.gen_erdos_renyi(n, p, seed + idx)))
            idx += 1
    for scale in (4, 6):
        for ef in (4, 8):
            nn, uv = port.gen_kronecker(scale, ef, seed + idx)
            out.append((f"kron{scale}_{ef}", nn, uv))
            idx += 1
    return out


def test_builder_matches_oracle_small(ssb, port):
    for name, n, uv in small_graphs(port):
        g = ssb.Graph.from_pairs(uv, n)
        row, col = port.to_csr(n, uv)
        for C_ in (1, 2, 3, 8, 32):
            for sig in (1, 2, 5, n):
                r = ssb.build_slimsell(g, C_, sig)
                L = port.build_slimsell(n, row, col, C_, sig)
                assert np.array_equal(r.col, L.col), (name, C_, sig)
                assert np.array_equal(r.cs, L.cs) and np.array_equal(r.cl, L.cl)
                assert np.array_equal(r.perm, L.perm) and r.padding == L.padding


# ---- kernel-level spmv_step -----------------------------------------------------

def test_spmv_step_golden(ssb, port, golden):
    r = ssb.build_slimsell(ssb.gen_kronecker(10, 16, 1), 8, 8)
    for c in golden["kron10_spmv_C8_s8"]:
        out = ssb.spmv_step(r, ssb.Variant(c["variant"]), np.array(c["x"], dtype=np.int64))
        assert port.fnv(out) == c["out_fnv"]


def test_spmv_step_random_vs_oracle(ssb, port):
    n, uv = port.gen_kronecker(9, 8, 3)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    rng = np.random.default_rng(0)
    for C_ in (1, 3, 8, 32):
        r = ssb.build_slimsell(g, C_, n)
        L = port.build_slimsell(n, row, col, C_, n)
        for v in range(4):
            x = rng.integers(-(1 << 40), 1 << 40, r.n_padded)
            if v == 0:
                x[rng.random(r.n_padded) < 0.5] = KINF
            cb, ce = 1, max(1, r.n_chunks - 1)
            base = rng.integers(0, 9, r.n_padded)
            a = ssb.spmv_step(r, ssb.Variant(v), x, base.copy(), cb, ce)
            b = port.spmv_step(L, v, x, base.copy(), cb, ce)
            assert np.array_equal(a, b), (C_, v)
    with pytest.raises(ssb.InvalidArgument):
        ssb.spmv_step(r, ssb.Variant.real, np.zeros(r.n_padded, np.int64), None, 0, r.n_chunks + 1)
    with pytest.raises(ssb.InvalidArgument):
        ssb.spmv_step(r, ssb.Variant.real, np.zeros(3, np.int64))


def test_spmv_split_hub_chunks_device_operands_and_segment(ssb, port):
    """Hub chunks longer than one work unit (1024 columns) are split and folded
    by atomics: the host form, the device-operand form (ssb_spmv_step_device)
    and the oracle agree for every semiring, C in {8, 32}; spmv_segment
    (repr.cpp:20-35) equals the reference loop restated on the oracle's layout,
    including column ranges crossing unit boundaries."""
    import torch
    n, uv = port.gen_kronecker(14, 32, 1)  # max degree > 1024
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    rng = np.random.default_rng(3)
    ops = {0: (lambda a, b: min(a, b), lambda a, b: KINF if KINF in (a, b) else a + b, KINF, 1, KINF),
           1: (lambda a, b: (a + b + (1 << 63)) % (1 << 64) - (1 << 63),
               lambda a, b: (a * b + (1 << 63)) % (1 << 64) - (1 << 63), 0, 1, 0),
           2: (lambda a, b: a | b, lambda a, b: a & b, 0, 1, 0),
           3: (lambda a, b: max(a, b), lambda a, b: (a * b + (1 << 63)) % (1 << 64) - (1 << 63), 0, 1, 0)}
    for C_ in (8, 32):
        r = ssb.build_slimsell(g, C_, n)
        L = port.build_slimsell(n, row, col, C_, n)
        assert int(L.cl.max()) > 1024
        for v in range(4):
            x = rng.integers(-(1 << 40), 1 << 40, r.n_padded)
            if v == 0:
                x[rng.random(r.n_padded) < 0.5] = KINF
            want = port.spmv_step(L, v, x)
            assert np.array_equal(ssb.spmv_step(r, ssb.Variant(v), x), want), (C_, v)
            dx = torch.from_numpy(x).cuda()
            dout = torch.zeros(r.n_padded, dtype=torch.int64, device="cuda")
            ms = ssb.spmv_step_device(r, ssb.Variant(v), dx, dout)
            assert ms >= 0 and np.array_equal(dout.cpu().numpy(), want), (C_, v)
            # spmv_segment on the hub chunk, a range crossing unit boundaries
            plus, times, zero, edge, pad = ops[v]
            ch = int(np.argmax(L.cl))
            for cb, ln in ((0, int(L.cl[ch])), (1000, 1100), (5, 0), (int(L.cl[ch]) - 3, 3)):
                acc0 = rng.integers(0, 50, C_)
                got = ssb.spmv_segment(r, ssb.Variant(v), x, acc0.copy(), ch, cb, ln)
                exp = [int(a) for a in acc0]
                for j in range(cb, cb + ln):
                    for lane in range(C_):
                        c = int(L.col[L.cs[ch] + j * C_ + lane])
                        exp[lane] = plus(exp[lane], times(int(x[max(c, 0)]), pad if c < 0 else edge))
                assert got.tolist() == exp, (C_, v, cb, ln)
        with pytest.raises(ssb.InvalidArgument):
            ssb.spmv_segment(r, ssb.Variant.real, x, np.zeros(C_, np.int64), 0, 0, int(L.cl[0]) + 1)
        with pytest.raises(ssb.InvalidArgument):
            ssb.spmv_segment(r, ssb.Variant.real, x, np.zeros(C_, np.int64), r.n_chunks, 0, 1)


# ---- BFS ------------------------------------------------------------------------

def test_selftest_grid_vs_oracle(ssb, port):
    """The reference selftest's oracle grid (cli.cpp:427-466) plus C=32 (the
    persistent engine): dist, parents and every counter equal the oracle."""
    count = 0
    for name, n, uv in small_graphs(port):
        g = ssb.Graph.from_pairs(uv, n)
        row, col = port.to_csr(n, uv)
        csr = ssb.to_csr(g)
        for C_ in (2, 8, 32):
            for sig in (1, n):
                r = ssb.build_slimsell(g, C_, sig)
                L = port.build_slimsell(n, row, col, C_, sig)
                for root in (0, n // 2):
                    for v in range(4):
                        for sw in (False, True):
                            for Lc in (0, 4):
                                a = ssb.bfs_spmv(r, root, opts(ssb, v, sw, Lc), csr)
                                b = port.bfs_spmv(L, root, v, sw, Lc, csr=(row, col))
                                key = (name, C_, sig, root, v, sw, Lc)
                                assert a.iterations == b.iterations, key
                                assert np.array_equal(a.dist, b.dist), key
                                assert np.array_equal(a.parent, b.parent), key
                                assert dev_rows(a) == port_rows(b.stats), key
                                count += 1
    assert count == 16 * 3 * 2 * 2 * 4 * 4


def test_edge_graphs_vs_oracle(ssb, port, edge_graphs):
    """One vertex, no edges, loops only, two components, ragged n around C = 32
    (the port is pinned to the reference on the same list in test_oracle.py):
    layout, dist, parents and every counter equal the oracle."""
    for name, n, uv in edge_graphs:
        g = ssb.Graph.from_pairs(uv, n)
        assert g.num_vertices() == n and np.array_equal(g.edges(), uv), name
        row, col = port.to_csr(n, uv)
        csr = ssb.to_csr(g)
        for C_, sig in ((1, 1), (8, n), (32, n), (32, 1)):
            r = ssb.build_slimsell(g, C_, sig)
            L = port.build_slimsell(n, row, col, C_, sig)
            assert np.array_equal(r.col, L.col) and np.array_equal(r.perm, L.perm), (name, C_, sig)
            for root in sorted({0, n // 2, n - 1}):
                for v in range(4):
                    for sw, Lc in ((False, 0), (True, 0), (True, 4)):
                        a = ssb.bfs_spmv(r, root, opts(ssb, v, sw, Lc), csr)
                        b = port.bfs_spmv(L, root, v, sw, Lc, csr=(row, col))
                        key = (name, C_, sig, root, v, sw, Lc)
                        assert a.iterations == b.iterations, key
                        assert np.array_equal(a.dist, b.dist), key
                        assert np.array_equal(a.parent, b.parent), key
                        assert dev_rows(a) == port_rows(b.stats), key


def test_cfg1_golden(ssb, port, golden):
    """Config 1: S16, C=8, σ=C, sel-max, the 16 pick_roots roots (4 isolated,
    10 not perm fixed points — the reference's parent encoding is active)."""
    r = ssb.build_slimsell(ssb.gen_kronecker(16, 16, 1), 8, 8)
    cases = [c for c in golden["cases"] if c["graph"] == "kron16" and c["C"] == 8]
    assert len(cases) == 48
    for c in cases:
        res = ssb.bfs_spmv(r, c["root"], opts(ssb, 3, c["slimwork"], c["L"]))
        assert res.iterations == c["iterations"]
        assert port.fnv(res.dist) == c["dist_fnv"], c
        assert port.fnv(res.parent) == c["parent_fnv"], c
        assert dev_rows(res) == c["stats"], c


@pytest.mark.parametrize("graph", ["kron16", "kron20", "kron22"])
def test_c32_golden_all_semirings(ssb, port, golden, graph):
    scale = int(graph[4:])
    g = ssb.gen_kronecker(scale, 16, 1)
    r = ssb.build_slimsell(g, 32, g.num_vertices())
    csr = ssb.to_csr(g)
    cases = [c for c in golden["cases"] if c["graph"] == graph and c["C"] == 32]
    assert cases
    for c in cases:
        res = ssb.bfs_spmv(r, c["root"], opts(ssb, c["variant"], c["slimwork"], c["L"]), csr)
        assert res.iterations == c["iterations"], c
        assert port.fnv(res.dist) == c["dist_fnv"], c
        assert port.fnv(res.parent) == c["parent_fnv"], c
        assert dev_rows(res) == c["stats"], c


def test_kron10_full_vectors(ssb, golden):
    g = ssb.gen_kronecker(10, 16, 1)
    csr = ssb.to_csr(g)
    reprs = {}
    for c in golden["kron10_full"]:
        key = (c["C"], c["sigma"])
        if key not in reprs:
            reprs[key] = ssb.build_slimsell(g, *key)
        res = ssb.bfs_spmv(reprs[key], c["root"], opts(ssb, c["variant"], True, 4), csr)
        assert res.dist.tolist() == c["dist"]
        assert res.parent.tolist() == c["parent"]
        assert dev_rows(res) == c["stats"]


def test_selmax_corrected_parents_closed_form(ssb, port):
    """selmax_compat=False: parent = perm[max inv_perm[u] over neighbours one
    level up], root self-parented."""
    n, uv = port.gen_kronecker(12, 16, 5)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    for C_, sig in ((32, n), (8, 8)):
        r = ssb.build_slimsell(g, C_, sig)
        inv = r.inv_perm
        for root in (0, 17, 1000):
            res = ssb.bfs_spmv(r, root, opts(ssb, 3, True, 16, compat=False))
            d = res.dist
            for v in range(n):
                if d[v] == KINF:
                    assert res.parent[v] == -1
                elif d[v] == 0:
                    assert res.parent[v] == v
                else:
                    nb = col[row[v]:row[v + 1]]
                    up = nb[d[nb] == d[v] - 1]
                    assert res.parent[v] == up[np.argmax(inv[up])]


def test_bfs_properties_large(ssb):
    """Size-independent BFS invariants at S22 (C=32): every edge spans at most
    one level, every reached non-root vertex has a parent one level up, the
    four semirings agree on dist, and counters add up."""
    g = ssb.gen_kronecker(22, 16, 2)
    r = ssb.build_slimsell(g, 32, g.num_vertices())
    uv = g.edges()
    dists = []
    for v in range(4):
        res = ssb.bfs_spmv(r, 123, opts(ssb, v, True, 128, compat=False))
        d = res.dist
        du, dv = d[uv[:, 0]], d[uv[:, 1]]
        both = (du != KINF) & (dv != KINF)
        assert np.all(np.abs(du[both] - dv[both]) <= 1)
        assert np.all((du == KINF) == (dv == KINF))
        for s in res.per_iter:
            assert s.chunks_processed + s.chunks_skipped == r.n_chunks
        assert sum(s.frontier_size for s in res.per_iter) == int(np.sum(d != KINF)) - 1
        if v == 3:
            p = res.parent
            reached = np.nonzero((d != KINF) & (d > 0))[0]
            assert np.all(d[p[reached]] == d[reached] - 1)
        dists.append(d)
    for d in dists[1:]:
        assert np.array_equal(d, dists[0])


def test_device_bfs_handle_and_traversed_edges(ssb, port):
    n, uv = port.gen_kronecker(14, 16, 1)
    g = ssb.Graph.from_pairs(uv, n)
    r = ssb.build_slimsell(g, 32, n)
    row, col = port.to_csr(n, uv)
    db = ssb.DeviceBfs(r)
    k, ms, stats, rc = db.run(5, opts(ssb, 3, True, 64))
    assert rc == 0 and ms > 0 and len(stats) == k
    dist, parent = db.fetch(True)
    b = port.bfs_spmv(port.build_slimsell(n, row, col, 32, n), 5, 3, True, 64)
    assert np.array_equal(dist, b.dist) and np.array_equal(parent, b.parent)
    deg = np.diff(row)
    assert db.edges_traversed() == int(deg[dist != KINF].sum() // 2)


def test_errors(ssb):
    g = ssb.gen_path(4)
    r = ssb.build_slimsell(g, 2, 1)
    with pytest.raises(ssb.OutOfRange):
        ssb.bfs_spmv(r, 4)
    with pytest.raises(ssb.OutOfRange):
        ssb.bfs_spmv(r, -1)
    with pytest.raises(ssb.InvalidArgument):
        ssb.build_slimsell(g, 0, 1)
    with pytest.raises(ssb.InvalidArgument):
        ssb.build_slimsell(g, 2, 0)
    for C_ in (2, 32):
        r = ssb.build_slimsell(g, C_, 1)
        with pytest.raises(ssb.BfsCapError) as ei:
            ssb.bfs_spmv(r, 0, opts(ssb, 0, max_it=2))
        assert ei.value.partial.dist.tolist() == [0, 1, 2, KINF]
        assert ei.value.partial.parent.size == 0 and ei.value.partial.iterations == 2
    # isolated root: one iteration, nothing reached
    g = ssb.Graph.from_pairs(np.array([[0, 1]]), 3)
    for C_ in (1, 32):
        res = ssb.bfs_spmv(ssb.build_slimsell(g, C_, 3), 2, opts(ssb, 3))
        assert res.iterations == 1 and res.dist.tolist() == [KINF, KINF, 0]
        assert res.parent.tolist() == [-1, -1, 2]


@pytest.mark.parametrize("mode_env", [
    {"SSB_DENSE_DIV": "1000000000"},   # always the sparse sweep
    {"SSB_DENSE_DIV": "1"},            # early-exit sweeps whenever |F| > 1
    {"SSB_DENSE_DIV": "4096"},         # the default switch point
    {"SSB_DENSE_DIV": "1000000000", "SSB_SUMMARY_SHIFT": "6"},  # 64-vertex summary, sparse
    {"SSB_DENSE_DIV": "1", "SSB_SUMMARY_SHIFT": "6"},           # 64-vertex summary, early exit
    # the hashed summary (built by sparse iterations, probed by the next
    # early-exit one), also carried across one-iteration launches
    {"SSB_DENSE_DIV": "4096", "SSB_SUMMARY_SHIFT": "8", "SSB_HASH_MIN_BITS": "1"},
    {"SSB_DENSE_DIV": "4096", "SSB_SUMMARY_SHIFT": "8", "SSB_HASH_MIN_BITS": "1",
     "SSB_ITERS_PER_LAUNCH": "1"},
    {"SSB_DENSE_DIV": "64", "SSB_SUMMARY_SHIFT": "8", "SSB_HASH_MIN_BITS": "1",
     "SSB_HASH_THR": "1000000000"},
])
def test_sweep_modes_with_small_shared_image(ssb, port, monkeypatch, mode_env):
    """Both sweep modes (sparse / early-exit) with a tiny shared-memory
    image, so the prefix + summary split and the tail paths are exercised at
    small scale, against the oracle (all semirings, SlimWork, SlimChunk)."""
    monkeypatch.setenv("SSB_SMEM_KB", "2")
    for k_, v_ in mode_env.items():
        monkeypatch.setenv(k_, v_)
    n, uv = port.gen_kronecker(14, 16, 9)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    csr = ssb.to_csr(g)
    r = ssb.build_slimsell(g, 32, n)
    L = port.build_slimsell(n, row, col, 32, n)
    for root in (0, 3, 777, 9000):
        for v in range(4):
            for sw, Lc in ((True, 16), (False, 0), (True, 0)):
                a = ssb.bfs_spmv(r, root, opts(ssb, v, sw, Lc), csr)
                b = port.bfs_spmv(L, root, v, sw, Lc, csr=(row, col))
                key = (root, v, sw, Lc)
                assert np.array_equal(a.dist, b.dist), key
                assert np.array_equal(a.parent, b.parent), key
                assert dev_rows(a) == port_rows(b.stats), key


@pytest.mark.parametrize("world", [1, 2, 3])
def test_chunk_sharded_device_bfs_matches_single_gpu(ssb, port, monkeypatch, world):
    """The multi-GPU decomposition (chunk-range shards + per-iteration frontier
    all-gather) run with `world` shards emulated on one GPU — separate device
    layouts and workspaces, stepped in lockstep, the all-gather done in-process
    — equals the reference (oracle) in dist, sel-max parents and counters."""
    from paper_2010_09913_b200.sharding import DeviceShard, LocalComm, partition_chunks, run_sharded_bfs
    monkeypatch.setenv("SSB_SMEM_KB", "4")  # exercise prefix + summary + exact lookups
    n, uv = port.gen_kronecker(15, 16, 2)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    reprs = [ssb.build_slimsell(g, 32, n) for _ in range(world)]
    ranges = partition_chunks(reprs[0].cl, 32, world)
    shards = [DeviceShard(r, b, e) for r, (b, e) in zip(reprs, ranges)]
    for root in (0, 5, 2000):
        for v, sw, Lc in ((3, True, 64), (0, True, 0), (3, False, 0), (1, True, 16)):
            o = opts(ssb, v, sw, Lc)
            dist, parent, per_iter = run_sharded_bfs(shards, LocalComm(), root, o)
            b = port.bfs_spmv(L, root, v, sw, Lc)
            assert np.array_equal(dist, b.dist), (root, v, world)
            if v == 3:
                assert np.array_equal(parent, b.parent), (root, v, world)
            assert dev_rows(ssb.BfsResult(dist, parent, len(per_iter), per_iter)) == port_rows(b.stats)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_chunk_sharded_async_steps_match_oracle(ssb, port, monkeypatch, world):
    """The NCCL form without host round trips (ssb_bfs_shard_*_async: the
    sweep reads |F|, the task list and the retired-chunk count from a device
    carry; the exchange counts |F| on the device; the host polls |F_{k-1}|
    while k is queued; counters summed once at the end). `world` shards, each
    on its own library stream, the all-gather done on a third stream with
    events between them — the ordering NCCL gives on one stream per rank —
    equal the oracle in dist, sel-max parents and every counter, including
    the iteration queued after convergence (a no-op) and the cap."""
    import torch

    from paper_2010_09913_b200.sharding import DeviceShard, LocalComm, partition_chunks, run_sharded_bfs_async
    monkeypatch.setenv("SSB_SMEM_KB", "4")
    n, uv = port.gen_kronecker(15, 16, 2)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    reprs = [ssb.build_slimsell(g, 32, n) for _ in range(world)]
    ranges = partition_chunks(reprs[0].cl, 32, world)
    shards = [DeviceShard(r, b, e) for r, (b, e) in zip(reprs, ranges)]
    side = torch.cuda.Stream()

    def run(root, o):
        for sh in shards:
            sh.begin_async(root, o)
        k, iters = 0, None
        while iters is None:
            k += 1
            owned, evs = [], []
            for sh in shards:
                with torch.cuda.stream(sh.stream()):
                    owned.append(sh.step_async())
                    evs.append(torch.cuda.Event())
                    evs[-1].record()
            with torch.cuda.stream(side):
                for e in evs:
                    side.wait_event(e)
                full = LocalComm().allgather_frontier(owned)
                done = torch.cuda.Event()
                done.record()
            for sh in shards:
                with torch.cuda.stream(sh.stream()):
                    sh.stream().wait_event(done)
                    sh.exchange_async(full)
            if k >= 2 and shards[0].front(k - 1) == 0:
                iters = k - 1
            assert all(sh.front(k) == shards[0].front(k) for sh in shards)
        parts = [sh.finish(iters)[0] for sh in shards]
        per = []
        for i in range(iters):
            f = lambda key: sum(getattr(p[i], key) for p in parts)  # noqa: E731
            per.append(ssb.IterStats(i + 1, 0, f("chunks_processed"), f("chunks_skipped"),
                                     f("subchunks_processed"), f("columns_processed"), f("frontier_size")))
        dist = np.full(n, KINF, np.int64)
        parent = np.full(n, -1, np.int64)
        for sh in shards:
            sh.fetch(o.variant == 3, dist, parent)
        return dist, parent, per

    for root in (0, 5, 2000):
        for v, sw, Lc in ((3, True, 64), (0, True, 0), (3, False, 0), (2, True, 2048)):
            o = opts(ssb, v, sw, Lc)
            dist, parent, per_iter = run(root, o)
            b = port.bfs_spmv(L, root, v, sw, Lc)
            assert np.array_equal(dist, b.dist), (root, v, world)
            if v == 3:
                assert np.array_equal(parent, b.parent), (root, v, world)
            assert dev_rows(ssb.BfsResult(dist, parent, len(per_iter), per_iter)) == port_rows(b.stats)
    if world == 1:  # the library driver itself (one rank, a device-side comm)
        class OneRank:
            device_async = True

            def allgather_frontier(self, owned_list):
                return owned_list[0]

            def allreduce_sum(self, arrays):
                return arrays[0]

        o = opts(ssb, 3, True, 64)
        for root in (0, 5, 2000):
            dist, parent, per_iter = run_sharded_bfs_async(shards[0], OneRank(), root, o)
            b = port.bfs_spmv(L, root, 3, True, 64)
            assert np.array_equal(dist, b.dist) and np.array_equal(parent, b.parent)
            assert dev_rows(ssb.BfsResult(dist, parent, len(per_iter), per_iter)) == port_rows(b.stats)
        o.max_iterations = 2
        with pytest.raises(ssb.BfsCapError) as ei:
            run_sharded_bfs_async(shards[0], OneRank(), 5, o)
        assert ei.value.partial.iterations == 2 and len(ei.value.partial.parent) == 0
        b = port.bfs_spmv(L, 5, 3, True, 64, max_iterations=2)
        assert np.array_equal(ei.value.partial.dist, b.dist)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_fused_p2p_sharded_bfs_matches_oracle(ssb, port, monkeypatch, world):
    """The fused multi-GPU BFS (frontier words stored into the peers' windows
    and a counter barrier inside the BFS kernel, ssb_bfs_p2p*) with `world`
    ranks emulated in ONE cooperative launch on this device — the same kernel
    and exchange code a multi-GPU job runs, peers being plain device memory —
    equals the reference (oracle) in dist, sel-max parents and counters, over
    repeated BFS on the same windows (barrier generations carry over)."""
    from paper_2010_09913_b200.sharding import partition_chunks, run_p2p_group
    monkeypatch.setenv("SSB_SMEM_KB", "4")  # prefix + summary + exact lookups; summary words shared at range ends
    n, uv = port.gen_kronecker(15, 16, 2)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    reprs = [ssb.build_slimsell(g, 32, n) for _ in range(world)]
    ranges = partition_chunks(reprs[0].cl, 32, world)
    for root in (0, 5, 2000, 31000):
        for v, sw, Lc in ((3, True, 64), (0, True, 0), (3, False, 0), (1, True, 16), (2, True, 2048)):
            o = opts(ssb, v, sw, Lc)
            dist, parent, per_iter, ms = run_p2p_group(reprs, ranges, root, o)
            b = port.bfs_spmv(L, root, v, sw, Lc)
            assert np.array_equal(dist, b.dist), (root, v, world)
            if v == 3:
                assert np.array_equal(parent, b.parent), (root, v, world)
            assert dev_rows(ssb.BfsResult(dist, parent, len(per_iter), per_iter)) == port_rows(b.stats)
    # an uneven split (one rank owns a single chunk) and the iteration cap
    nc = reprs[0].n_chunks
    odd = [(0, 1), (1, nc)] + [(nc, nc)] * (world - 2)
    o = opts(ssb, 3, True, 64)
    dist, parent, _, _ = run_p2p_group(reprs, odd, 5, o)
    b = port.bfs_spmv(L, 5, 3, True, 64)
    assert np.array_equal(dist, b.dist) and np.array_equal(parent, b.parent)
    o.max_iterations = 2
    with pytest.raises(ssb.DeviceError):
        run_p2p_group(reprs, ranges, 5, o)
    o.max_iterations = 0
    dist, _, _, _ = run_p2p_group(reprs, ranges, 5, o)  # usable after a capped BFS
    assert np.array_equal(dist, b.dist)


def test_fused_p2p_default_geometry_matches_single_gpu(ssb):
    """The emulated fused multi-GPU BFS at S20 with the production image
    geometry (160 KB: prefix + summary, dense/direct probe modes all reached)
    equals the single-GPU engine bit for bit, counters included."""
    from paper_2010_09913_b200.sharding import partition_chunks, run_p2p_group
    g = ssb.gen_kronecker(20, 16, 1)
    n = g.num_vertices()
    reprs = [ssb.build_slimsell(g, 32, n) for _ in range(4)]
    for world in (3, 4):
        ranges = partition_chunks(reprs[0].cl, 32, world)
        for root in (0, 12345, 777777):
            for v in (3, 0):
                o = opts(ssb, v, True, 256)
                a = ssb.bfs_spmv(reprs[0], root, o)
                dist, parent, per_iter, _ = run_p2p_group(reprs[:world], ranges, root, o)
                assert np.array_equal(dist, a.dist), (world, root, v)
                if v == 3:
                    assert np.array_equal(parent, a.parent), (world, root, v)
                assert dev_rows(ssb.BfsResult(dist, parent, len(per_iter), per_iter)) == dev_rows(a)


@pytest.mark.parametrize("world", [2, 3])
def test_range_built_shards(ssb, port, world):
    """ssb_build_slimsell_range: every rank holds only its own chunks' cells
    (SURVEY.md §8(e)). The cells equal the matching slice of the whole layout,
    perm / cl / degrees equal the whole layout's, whole-layout calls are
    refused, and the fused and the host-driven sharded BFS over range-built
    handles equal the single-GPU result."""
    from paper_2010_09913_b200.sharding import (DeviceShard, LocalComm, partition_chunks, run_p2p_group,
                                                run_sharded_bfs)
    g = ssb.gen_kronecker(18, 16, 4)
    n = g.num_vertices()
    full = ssb.build_slimsell(g, 32, n)
    ranges = partition_chunks(full.cl, 32, world)
    col = full.col32()
    cs = full.cs
    parts = [ssb.build_slimsell(g, 32, n, chunk_range=rg) for rg in ranges]
    for (b, e), r in zip(ranges, parts):
        assert (r.range_begin, r.range_end) == (b, e) and r.n_cells == full.n_cells
        lo = int(cs[b]) if b < full.n_chunks else full.n_cells
        hi = int(cs[e]) if e < full.n_chunks else full.n_cells
        assert np.array_equal(r.col32(), col[lo:hi]), (b, e)
        assert np.array_equal(r.cl, full.cl) and np.array_equal(r.perm, full.perm)
        assert np.array_equal(r.degrees(), full.degrees())
        if r.partial:
            with pytest.raises(ssb.InvalidArgument):
                ssb.bfs_spmv(r, 0, opts(ssb, 3))
            with pytest.raises(ssb.InvalidArgument):
                r.col
    shards = [DeviceShard(r, b, e) for r, (b, e) in zip(parts, ranges)]
    for root in (0, 1000, 200000):
        for v in (3, 0):
            o = opts(ssb, v, True, 512)
            a = ssb.bfs_spmv(full, root, o)
            d1, p1, it1, _ = run_p2p_group(parts, ranges, root, o)
            d2, p2, it2 = run_sharded_bfs(shards, LocalComm(), root, o)
            for d, p, it in ((d1, p1, it1), (d2, p2, it2)):
                assert np.array_equal(d, a.dist), (world, root, v)
                if v == 3:
                    assert np.array_equal(p, a.parent), (world, root, v)
                assert dev_rows(ssb.BfsResult(d, p, len(it), it)) == dev_rows(a)


@pytest.mark.parametrize("world,k", [(2, 3), (3, 2), (4, 4), (8, 4)])
def test_round_robin_segment_shards(ssb, world, k):
    """Ranks owning k round-robin (snake-dealt) chunk segments each, built
    with only those segments' cells (ssb_build_slimsell_segments): the cells
    are the matching slices of the whole layout in order, and the fused BFS
    over them (segments exchanged separately, summary words shared at every
    segment end) equals the single-GPU result."""
    from paper_2010_09913_b200.sharding import partition_segments, run_p2p_group
    g = ssb.gen_kronecker(18, 16, 8)
    n = g.num_vertices()
    full = ssb.build_slimsell(g, 32, n)
    segs = partition_segments(full.cl, 32, world, k)
    assert sorted(x for sg in segs for x in sg) == [tuple(x) for x in
                                                    __import__("paper_2010_09913_b200.sharding", fromlist=["x"])
                                                    .partition_chunks(full.cl, 32, world * k)]
    col, cs = full.col32(), np.concatenate([full.cs, [full.n_cells]])
    parts = [ssb.build_slimsell(g, 32, n, segments=sg) for sg in segs]
    for sg, r in zip(segs, parts):
        want = np.concatenate([col[cs[b]:cs[e]] for b, e in sg if e > b] or [col[:0]])
        assert np.array_equal(r.col32(), want)
    for root in (0, 4321, 150000):
        for v in (3, 1):
            o = opts(ssb, v, True, 256)
            a = ssb.bfs_spmv(full, root, o)
            d, p, it, _ = run_p2p_group(parts, segs, root, o)
            assert np.array_equal(d, a.dist), (world, k, root, v)
            if v == 3:
                assert np.array_equal(p, a.parent), (world, k, root, v)
            assert dev_rows(ssb.BfsResult(d, p, len(it), it)) == dev_rows(a)


def test_multi_pass_build_equals_single_pass(ssb, monkeypatch):
    """The builder sorts and scatters arcs in passes over row sub-ranges when
    2m arcs do not fit beside col (S28 on one B200); forced to many small
    passes it must produce the identical layout, whole and range-built."""
    g = ssb.gen_kronecker(17, 16, 6)
    n = g.num_vertices()
    ref = ssb.build_slimsell(g, 32, n)
    col, cl, perm = ref.col32(), ref.cl, ref.perm
    monkeypatch.setenv("SSB_ARCS_PER_PASS", "50000")
    r = ssb.build_slimsell(g, 32, n)
    assert np.array_equal(r.col32(), col) and np.array_equal(r.cl, cl) and np.array_equal(r.perm, perm)
    b, e = 100, ref.n_chunks - 77
    part = ssb.build_slimsell(g, 32, n, chunk_range=(b, e))
    assert np.array_equal(part.col32(), col[int(ref.cs[b]): int(ref.cs[e])])
    r8 = ssb.build_slimsell(g, 8, 8)
    # the validator's / queue BFS's device CSR is built in passes the same way
    g2 = ssb.gen_kronecker(17, 16, 6)
    t_multi = ssb.bfs_traditional(g2, 3)
    monkeypatch.delenv("SSB_ARCS_PER_PASS")
    assert np.array_equal(r8.col32(), ssb.build_slimsell(g, 8, 8).col32())
    t_one = ssb.bfs_traditional(g, 3)
    assert np.array_equal(t_multi.dist, t_one.dist) and np.array_equal(t_multi.parent, t_one.parent)
    assert ssb.validate_bfs(g2, 3, t_one.dist, t_one.parent) is None


def test_fused_p2p_rank_path_world1(ssb, port, monkeypatch):
    """The per-rank entry points a multi-GPU job uses (ssb_p2p_window → IPC
    handle, ssb_p2p_attach, ssb_bfs_p2p with the one-launch-per-rank kernel,
    ssb_bfs_shard_fetch) at world 1: the exchange has no peers but the kernel,
    its barrier generations and the window reset run exactly as on a rank."""
    from paper_2010_09913_b200.sharding import P2PShard
    monkeypatch.setenv("SSB_SMEM_KB", "4")
    n, uv = port.gen_kronecker(14, 16, 5)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    r = ssb.build_slimsell(g, 32, n)
    sh = P2PShard(r, 0, r.n_chunks)
    h = sh.window_handle()
    assert len(h) == 64
    sh.attach(0, 1, [h])
    for root in (0, 17, 9000):
        for v in (3, 0):
            o = opts(ssb, v, True, 64)
            k, ms, st = sh.run(root, o)
            dist = np.full(n, ssb.KINF, np.int64)
            parent = np.full(n, -1, np.int64)
            sh.fetch(v == 3, dist, parent)
            b = port.bfs_spmv(L, root, v, True, 64)
            assert np.array_equal(dist, b.dist), (root, v)
            if v == 3:
                assert np.array_equal(parent, b.parent), (root, v)
            assert dev_rows(ssb.BfsResult(dist, parent, k, st)) == port_rows(b.stats)


def test_fetch_wire_format_equals_direct_path(ssb, port, monkeypatch):
    """Whole-result fetches go through the narrow wire format (uint8 levels +
    int32 parents over PCIe — or, for sel-max, one packed 32-bit word of level
    and parent id — widened to int64 by host threads); it must equal
    the direct int64 path (SSB_WIRE=0) and the oracle, into pageable and
    pinned outputs, for sel-max parents and dp_transform parents, and with the
    chunking pushed to odd sizes."""
    import torch
    n, uv = port.gen_kronecker(17, 16, 3)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    r = ssb.build_slimsell(g, 32, n)
    csr = ssb.to_csr(g)
    pin_d = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    pin_p = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    for root in (0, 4242):
        for v in (3, 0, 2):
            o = opts(ssb, v, True, 64)
            b = port.bfs_spmv(L, root, v, True, 64, csr=(row, col))
            outs = []
            # (sel-max with dist and parents: the packed 4-byte wire by
            # default, the 5-byte one with SSB_WIRE_PACKED=0)
            for wire, chunks, packed in (("1", "16", "1"), ("1", "7", "1"), ("1", "16", "0"), ("0", "16", "1")):
                monkeypatch.setenv("SSB_WIRE", wire)
                monkeypatch.setenv("SSB_WIRE_CHUNKS", chunks)
                monkeypatch.setenv("SSB_WIRE_PACKED", packed)
                a = ssb.bfs_spmv(r, root, o, csr)
                pin_d.fill(-7)
                pin_p.fill(-7)
                c = ssb.bfs_spmv(r, root, o, csr, pin_d, pin_p)
                outs.append((a.dist.copy(), a.parent.copy(), c.dist.copy(), c.parent.copy()))
                # outputs whose addresses differ by 8 bytes mod 32 (no common
                # alignment for streaming stores)
                md = np.full(n, -7, np.int64)
                mp = np.full(n + 1, -7, np.int64)[1:]
                e = ssb.bfs_spmv(r, root, o, csr, md, mp)
                outs.append((e.dist.copy(), e.parent.copy(), md.copy(), mp.copy()))
            for d1, p1, d2, p2 in outs:
                assert np.array_equal(d1, b.dist) and np.array_equal(d2, b.dist), (root, v)
                assert np.array_equal(p1, b.parent) and np.array_equal(p2, b.parent), (root, v)


def test_bfs_spmv_batch_equals_single_calls(ssb, port):
    """ssb_bfs_spmv_batch (root i's fetch overlapped with root i+1's BFS, two
    wire slots) delivers exactly what per-root ssb_bfs_spmv calls deliver —
    sel-max parents, dp_transform parents with a CSR, aliased output buffers
    (the last root's result survives), the small-graph direct path, and the
    iteration cap (the capped root's dist delivered, its index reported)."""
    import torch
    for scale in (17, 10):
        n, uv = port.gen_kronecker(scale, 16, 2)
        g = ssb.Graph.from_pairs(uv, n)
        r = ssb.build_slimsell(g, 32, n)
        csr = ssb.to_csr(g)
        roots = [0, 77, 5, n - 1, 123]
        for v, c in ((3, None), (0, csr), (2, None)):
            o = opts(ssb, v, True, 64)
            ref = [ssb.bfs_spmv(r, x, o, c) for x in roots]
            ds = [np.full(n, -9, np.int64) for _ in roots]
            ps = [np.full(n, -9, np.int64) for _ in roots]
            its = ssb.bfs_spmv_batch(r, roots, o, c, ds, ps)
            assert its == [x.iterations for x in ref]
            for a, d, p in zip(ref, ds, ps):
                assert np.array_equal(a.dist, d), (scale, v)
                if len(a.parent):
                    assert np.array_equal(a.parent, p), (scale, v)
            # aliased pinned outputs: the last root's result remains
            pd = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
            pp = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
            ssb.bfs_spmv_batch(r, roots, o, c, [pd] * len(roots), [pp] * len(roots))
            assert np.array_equal(pd, ref[-1].dist)
            if len(ref[-1].parent):
                assert np.array_equal(pp, ref[-1].parent)
    o = opts(ssb, 3, True, 64, max_it=2)
    with pytest.raises(ssb.BfsCapError) as ei:
        ssb.bfs_spmv_batch(r, [0, 5], o)
    assert ei.value.root_index == 0
    with pytest.raises(ssb.OutOfRange):
        ssb.bfs_spmv_batch(r, [0, n], opts(ssb, 3))


def test_device_erdos_renyi_matches_oracle(ssb, port):
    """gen_erdos_renyi (generator.cpp:15-58) bit-exact, incl. p = 0 / 1 and
    the config-4 shape (average degree 16) at 2^18 and 2^20 vertices."""
    cases = [(1, 0.5, 1), (2, 1.0, 3), (50, 0.0, 3), (40, 1.0, 2), (300, 0.05, 7), (5000, 0.003, 11),
             (1 << 18, 16 / ((1 << 18) - 1), 1), (1 << 20, 16 / ((1 << 20) - 1), 1)]
    for n, p, seed in cases:
        g = ssb.gen_erdos_renyi(n, p, seed)
        nn, uv = port.gen_erdos_renyi(n, p, seed)
        assert g.num_vertices() == nn == n, (n, p, seed)
        assert np.array_equal(g.edges(), uv), (n, p, seed)
    with pytest.raises(ssb.InvalidArgument):
        ssb.gen_erdos_renyi(10, 1.5, 1)


def test_erdos_renyi_bfs_matches_oracle(ssb, port, monkeypatch):
    """A low-skew graph (config 4 shape at 2^16, with a 4 KB shared image so
    the prefix holds few cell targets): the engine picks the fine 64-vertex
    summary there; all semirings equal the oracle."""
    monkeypatch.setenv("SSB_SMEM_KB", "4")
    n = 1 << 16
    g = ssb.gen_erdos_renyi(n, 16 / (n - 1), 5)
    nn, uv = port.gen_erdos_renyi(n, 16 / (n - 1), 5)
    row, col = port.to_csr(nn, uv)
    r = ssb.build_slimsell(g, 32, n)
    L = port.build_slimsell(n, row, col, 32, n)
    csr = ssb.to_csr(g)
    for root in (0, 12345):
        for v in range(4):
            a = ssb.bfs_spmv(r, root, opts(ssb, v, True, 64), csr)
            b = port.bfs_spmv(L, root, v, True, 64, csr=(row, col))
            assert np.array_equal(a.dist, b.dist), (root, v)
            assert np.array_equal(a.parent, b.parent), (root, v)
            assert dev_rows(a) == port_rows(b.stats), (root, v)


def test_deep_bfs_spans_launches(ssb, port):
    """A BFS deeper than one cooperative launch (1024 iterations: a path of
    2600 vertices) carries its active task list, retired chunks and counters
    across launches, and its levels (> 254) take the direct int64 fetch —
    per call and in a batch — equal to the oracle."""
    n, uv = port.gen_path(2600)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    r = ssb.build_slimsell(g, 32, n)
    L = port.build_slimsell(n, row, col, 32, n)
    csr = ssb.to_csr(g)
    for root in (0, 1300):
        for v, sw, Lc in ((3, True, 64), (0, True, 0), (2, False, 16)):
            o = opts(ssb, v, sw, Lc)
            a = ssb.bfs_spmv(r, root, o, csr)
            b = port.bfs_spmv(L, root, v, sw, Lc, csr=(row, col))
            assert a.iterations == b.iterations > 1024 or root == 1300, (root, v)
            assert np.array_equal(a.dist, b.dist) and np.array_equal(a.parent, b.parent), (root, v)
            assert dev_rows(a) == port_rows(b.stats), (root, v)
            d = [np.empty(n, np.int64)]
            p = [np.empty(n, np.int64)]
            its = ssb.bfs_spmv_batch(r, [root], o, csr, d, p)
            assert its == [b.iterations] and np.array_equal(d[0], b.dist) and np.array_equal(p[0], b.parent)


def test_device_bfs_traditional_matches_oracle(ssb, port):
    """The device queue BFS (bfs.cpp:248-291) equals the oracle's bfs_traditional:
    dist, smallest-id parents and per-level frontier sizes."""
    for make, roots in ((lambda: port.gen_kronecker(14, 16, 3), (0, 5, 4000)),
                        (lambda: (2000, port.gen_path(2000)[1]), (0, 1999, 777)),
                        (lambda: port.gen_erdos_renyi(3000, 0.002, 4), (1, 2999))):
        n, uv = make()
        g = ssb.Graph.from_pairs(uv, n)
        row, col = port.to_csr(n, uv)
        for root in roots:
            a = ssb.bfs_traditional(g, root)
            bd, bp, bk = port.bfs_traditional(n, row, col, root)
            assert np.array_equal(a.dist, bd), root
            assert np.array_equal(a.parent, bp), root
            assert a.iterations == bk, root
    with pytest.raises(ssb.OutOfRange):
        ssb.bfs_traditional(g, -1)


def test_device_validator(ssb, port):
    """validate_bfs accepts correct BFS trees (device queue BFS, SpMV BFS with
    corrected sel-max parents, compat parents with the compat flag) and reports
    every kind of corruption."""
    n, uv = port.gen_kronecker(14, 16, 5)
    g = ssb.Graph.from_pairs(uv, n)
    r = ssb.build_slimsell(g, 32, n)
    deg = np.bincount(uv.ravel(), minlength=n)
    deg[0] = 0  # vertex 0 sits at position 0: the sel-max quirk would be invisible
    root = int(np.argmax(deg))
    t = ssb.bfs_traditional(g, root)
    assert ssb.validate_bfs(g, root, t.dist, t.parent) is None
    s = ssb.bfs_spmv(r, root, opts(ssb, 3, True, 64, compat=False))
    assert ssb.validate_bfs(g, root, s.dist, s.parent) is None
    c = ssb.bfs_spmv(r, root, opts(ssb, 3, True, 64, compat=True))
    assert ssb.validate_bfs(g, root, c.dist, c.parent, selmax_compat=True) is None
    rep = ssb.validate_bfs(g, root, c.dist, c.parent)  # the reference's own selftest failure
    assert rep is not None and "self-parented" in rep
    assert ssb.validate_bfs(g, root, t.dist) is None  # distances only
    reached = np.nonzero((t.dist != ssb.KINF) & (t.dist > 1))[0]
    v = int(reached[0])
    bad = t.parent.copy(); bad[v] = v
    assert "not a neighbor" in ssb.validate_bfs(g, root, t.dist, bad)
    d2 = t.dist.copy(); d2[v] += 2
    assert ssb.validate_bfs(g, root, d2, None) is not None
    un = np.nonzero(t.dist == ssb.KINF)[0]
    if len(un):
        p2 = t.parent.copy(); p2[int(un[0])] = root
        assert "unreached but parent set" in ssb.validate_bfs(g, root, t.dist, p2)
    d3 = t.dist.copy(); d3[v] = ssb.KINF
    assert "reached and an unreached" in ssb.validate_bfs(g, root, d3, None)


def test_ingest_to_device_graph(ssb, port):
    """Graph.from_edge_list / from_matrix_market: host parse + device
    normalisation equal the oracle's from_pairs of the same records; errors
    surface as the reference's exception kinds."""
    rng = np.random.default_rng(3)
    uv = rng.integers(0, 500, size=(3000, 2))
    text = "H 600 3000\n" + "\n".join(f"{u} {v}" for u, v in uv) + "\n"
    g = ssb.Graph.from_edge_list(text)
    n, ref_uv = port.from_pairs(uv, 600)
    assert g.num_vertices() == n == 600 and np.array_equal(g.edges(), ref_uv)
    mm = "%%MatrixMarket matrix coordinate pattern symmetric\n500 500 3000\n" + \
         "\n".join(f"{u + 1} {v + 1}" for u, v in uv) + "\n"
    g2 = ssb.Graph.from_matrix_market(mm)
    n2, ref2 = port.from_pairs(np.concatenate([uv, uv[:, ::-1]]), 500)
    assert g2.num_vertices() == n2 and np.array_equal(g2.edges(), ref2)
    r = ssb.build_slimsell(g2, 32, n2)
    assert ssb.bfs_spmv(r, int(uv[0, 0]), opts(ssb, 3, True, 16)).dist[int(uv[0, 0])] == 0
    with pytest.raises(ssb.ParseError) as e:
        ssb.Graph.from_edge_list("0 1\n1 2 3\n")
    assert e.value.line == 2
    with pytest.raises(ssb.InvalidArgument):
        ssb.Graph.from_edge_list("0 1\n", reject_asymmetric=True)
    with pytest.raises(ssb.OutOfRange):
        ssb.Graph.from_edge_list("H 2 1\n0 5\n")


def test_edge_graphs_batch_equals_single_calls(ssb, edge_graphs):
    """ssb_bfs_spmv_batch on the edge graphs (one vertex, no edges, ragged n):
    every root class, every semiring, the same results as per-root calls."""
    for name, n, uv in edge_graphs:
        g = ssb.Graph.from_pairs(uv, n)
        r = ssb.build_slimsell(g, 32, n)
        csr = ssb.to_csr(g)
        roots = sorted({0, n // 2, n - 1})
        for v in range(4):
            o = opts(ssb, v, True, 4)
            c = csr if v in (0, 1) else None
            ref = [ssb.bfs_spmv(r, x, o, c) for x in roots]
            ds = [np.full(n, -9, np.int64) for _ in roots]
            ps = [np.full(n, -9, np.int64) for _ in roots]
            assert ssb.bfs_spmv_batch(r, roots, o, c, ds, ps) == [x.iterations for x in ref], name
            for a, d, p in zip(ref, ds, ps):
                assert np.array_equal(a.dist, d), (name, v)
                if len(a.parent):
                    assert np.array_equal(a.parent, p), (name, v)


@pytest.mark.parametrize("world", [2, 3])
def test_edge_graphs_sharded_paths(ssb, port, edge_graphs, world):
    """The edge graphs through both multi-GPU decompositions (chunk-range
    shards + all-gather, and the fused peer-window kernel), emulated on one
    GPU: ranks owning no chunk (n = 1, n ≤ 64), ragged last chunks, no edges."""
    from paper_2010_09913_b200.sharding import (DeviceShard, LocalComm, partition_chunks,
                                                 run_p2p_group, run_sharded_bfs)
    for name, n, uv in edge_graphs:
        g = ssb.Graph.from_pairs(uv, n)
        row, col = port.to_csr(n, uv)
        L = port.build_slimsell(n, row, col, 32, n)
        reprs = [ssb.build_slimsell(g, 32, n) for _ in range(world)]
        ranges = partition_chunks(reprs[0].cl, 32, world)
        shards = [DeviceShard(r, b, e) for r, (b, e) in zip(reprs, ranges)]
        for root in sorted({0, n // 2, n - 1}):
            for v, sw, Lc in ((3, True, 4), (0, True, 0), (2, False, 0)):
                o = opts(ssb, v, sw, Lc)
                b = port.bfs_spmv(L, root, v, sw, Lc)
                for how in ("allgather", "p2p"):
                    if how == "allgather":
                        dist, parent, per_iter = run_sharded_bfs(shards, LocalComm(), root, o)
                    else:
                        dist, parent, per_iter, _ = run_p2p_group(reprs, ranges, root, o)
                    key = (name, how, root, v, world)
                    assert np.array_equal(dist, b.dist), key
                    if v == 3:
                        assert np.array_equal(parent, b.parent), key
                    assert dev_rows(ssb.BfsResult(dist, parent, len(per_iter), per_iter)) == port_rows(b.stats), key


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0]])
def test_single_process_context_matches_single_gpu(ssb, port, devices):
    """ssb_ctx_create / ssb_ctx_build / ssb_sharded_bfs: one host process
    driving a sharded layout (round-robin segments, each rank holding only
    its cells). On one B200 the ranks share device 0 and run as one
    cooperative launch; the results equal the single-GPU engine and the
    oracle in dist, sel-max parents and every counter."""
    from paper_2010_09913_b200.sharding import Context
    n, uv = port.gen_kronecker(16, 16, 3)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    ctx = Context(devices)
    sh = ctx.build(g, 32, n, segments=3)
    assert sum(sh.cells_per_rank) == L.n_cells and len(sh.cells_per_rank) == len(devices)
    for root in (0, 9, 40000):
        for v, sw, Lc in ((3, True, 64), (0, True, 0), (2, False, 2048)):
            o = opts(ssb, v, sw, Lc)
            res = sh.bfs_spmv(root, o)
            b = port.bfs_spmv(L, root, v, sw, Lc)
            assert np.array_equal(res.dist, b.dist), (root, v, devices)
            if v == 3:
                assert np.array_equal(res.parent, b.parent), (root, v, devices)
            else:
                assert len(res.parent) == 0
            assert dev_rows(res) == port_rows(b.stats), (root, v, devices)
    o = opts(ssb, 3, True, 64)
    o.max_iterations = 2
    with pytest.raises(ssb.BfsCapError):
        sh.bfs_spmv(0, o)
    with pytest.raises(ssb.OutOfRange):
        sh.bfs_spmv(n, opts(ssb, 3, True, 64))
    res = sh.bfs_spmv(9, opts(ssb, 3, True, 64))  # usable after the errors
    assert np.array_equal(res.dist, port.bfs_spmv(L, 9, 3, True, 64).dist)


def test_context_rejects_bad_device_lists(ssb):
    import torch

    from paper_2010_09913_b200.sharding import Context
    nd = torch.cuda.device_count()
    with pytest.raises(ssb.InvalidArgument):
        Context([nd])  # not present
    with pytest.raises(ssb.InvalidArgument):
        Context([0] * 9)  # more than 8 ranks
    if nd >= 2:
        with pytest.raises(ssb.InvalidArgument):
            Context([0, 0, 1])  # mixed


def test_spmv_step_on_range_built_handles(ssb, port):
    """spmv_step / spmv_step_device on a handle that holds only a chunk range
    (a multi-GPU rank's cells): the rows of that range equal the whole
    layout's product; ranges outside the held cells are refused."""
    import torch
    n, uv = port.gen_kronecker(13, 16, 4)
    g = ssb.Graph.from_pairs(uv, n)
    full = ssb.build_slimsell(g, 32, n)
    nc = full.n_chunks
    rng = np.random.default_rng(11)
    for b, e in ((0, nc // 3), (nc // 3, nc), (5, 6)):
        part = ssb.build_slimsell(g, 32, n, chunk_range=(b, e))
        for v in range(4):
            x = rng.integers(0, 1 << 30, full.n_padded)
            want = ssb.spmv_step(full, ssb.Variant(v), x, np.zeros(full.n_padded, np.int64), b, e)
            got = ssb.spmv_step(part, ssb.Variant(v), x, np.zeros(full.n_padded, np.int64), b, e)
            assert np.array_equal(got, want), (b, e, v)
            dx = torch.from_numpy(x).cuda()
            dout = torch.zeros(full.n_padded, dtype=torch.int64, device="cuda")
            ssb.spmv_step_device(part, ssb.Variant(v), dx, dout, b, e)
            assert np.array_equal(dout.cpu().numpy(), want), (b, e, v)
        if e < nc:
            with pytest.raises(ssb.InvalidArgument):
                ssb.spmv_step(part, ssb.Variant.real, x, None, b, e + 1)


@pytest.mark.parametrize("segments", [1, 8])
def test_context_segment_counts(ssb, port, segments):
    """ssb_ctx_build with 1 and 8 round-robin segments per rank (the two
    ends of the partition's range) equals the oracle."""
    from paper_2010_09913_b200.sharding import Context
    n, uv = port.gen_kronecker(14, 16, 6)
    g = ssb.Graph.from_pairs(uv, n)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 32, n)
    sh = Context([0, 0, 0]).build(g, 32, n, segments=segments)
    assert all(s <= segments for s in sh.segments_per_rank)
    for root in (1, 777):
        res = sh.bfs_spmv(root, opts(ssb, 3, True, 128))
        b = port.bfs_spmv(L, root, 3, True, 128)
        assert np.array_equal(res.dist, b.dist) and np.array_equal(res.parent, b.parent)
        assert dev_rows(res) == port_rows(b.stats)
