"""CPU suite: pins the oracle (plain-C restatement, oracle/slimsell_oracle.c)
against the reference's golden vectors, SPEC.md's hand-derived KATs and —
where oracle/_ref is built — the reference library itself."""
import numpy as np
import pytest

from oracle import BOOLEAN, KINF, REAL, SELMAX, TROPICAL

STAT_COLS = [0, 2, 3, 4, 5, 6]  # drop elapsed_ns


def rows(stats):
    return [[int(r[c]) for c in STAT_COLS] for r in stats]


# ---- graph + layout fingerprints (reference-generated) ----------------------

@pytest.mark.parametrize("scale", [10, 16])
def test_generator_and_layout_fingerprints(port, golden, scale):
    e = next(g for g in golden["graphs"] if g["scale"] == scale)
    n, uv = port.gen_kronecker(scale, 16, 1)
    assert (n, uv.shape[0]) == (e["n"], e["m"])
    assert port.fnv(uv) == e["edges_fnv"]
    row, col = port.to_csr(n, uv)
    for lay in e["layouts"]:
        L = port.build_slimsell(n, row, col, lay["C"], lay["sigma_in"])
        assert L.sigma == lay["sigma"] and L.n_cells == lay["n_cells"] and L.padding == lay["padding"]
        assert port.fnv(L.col) == lay["col_fnv"]
        assert port.fnv(L.cs) == lay["cs_fnv"]
        assert port.fnv(L.cl) == lay["cl_fnv"]
        assert port.fnv(L.perm) == lay["perm_fnv"]


def test_pick_roots_cfg1(port, golden):
    # cli.cpp:114-134 stream; SURVEY.md §8(c).6 lists the same 16 roots
    assert [int(r) for r in port.pick_roots(65536, 16, 1)] == golden["cfg1_roots"]
    assert golden["cfg1_roots"][:3] == [48515, 8361, 60807]


def test_cfg1_selmax_golden(port, golden):
    """Config 1 (S16, C=8, σ=C, sel-max, 16 roots) — dist, quirk parents, counters."""
    n, uv = port.gen_kronecker(16, 16, 1)
    row, col = port.to_csr(n, uv)
    L8 = port.build_slimsell(n, row, col, 8, 8)
    cases = [c for c in golden["cases"] if c["graph"] == "kron16" and c["C"] == 8]
    assert len(cases) == 48
    for c in cases:
        out = port.bfs_spmv(L8, c["root"], c["variant"], c["slimwork"], c["L"])
        assert out.iterations == c["iterations"]
        assert port.fnv(out.dist) == c["dist_fnv"], c
        assert port.fnv(out.parent) == c["parent_fnv"], c
        assert rows(out.stats) == c["stats"], c


def test_kron10_full_vectors(port, golden):
    n, uv = port.gen_kronecker(10, 16, 1)
    row, col = port.to_csr(n, uv)
    lays = {}
    for c in golden["kron10_full"]:
        key = (c["C"], c["sigma"])
        if key not in lays:
            lays[key] = port.build_slimsell(n, row, col, *key)
        out = port.bfs_spmv(lays[key], c["root"], c["variant"], True, 4, csr=(row, col))
        assert out.iterations == c["iterations"]
        assert out.dist.tolist() == c["dist"]
        assert out.parent.tolist() == c["parent"]
        assert rows(out.stats) == c["stats"]


def test_spmv_step_golden(port, golden):
    n, uv = port.gen_kronecker(10, 16, 1)
    row, col = port.to_csr(n, uv)
    L = port.build_slimsell(n, row, col, 8, 8)
    for c in golden["kron10_spmv_C8_s8"]:
        out = port.spmv_step(L, c["variant"], np.array(c["x"], dtype=np.int64))
        assert port.fnv(out) == c["out_fnv"]


# ---- SPEC.md hand-derived known answers ----------------

def path4(port):
    n, uv = port.from_pairs(np.array([[0, 1], [1, 2], [2, 3]]), 4)
    return n, uv, port.to_csr(n, uv)


def test_spec_layout_kats(port):
    n, uv, (row, col) = path4(port)
    assert row.tolist() == [0, 1, 3, 5, 6] and col.tolist() == [1, 0, 2, 1, 3, 2]  # test_graph.cpp:93-98
    L = port.build_slimsell(n, row, col, 2, 1)
    assert L.cs.tolist() == [0, 4] and L.cl.tolist() == [2, 2]
    assert L.col.tolist() == [1, 0, -1, 2, 1, 2, 3, -1] and L.padding == 2
    L = port.build_slimsell(n, row, col, 2, 4)
    assert L.perm.tolist() == [1, 2, 0, 3] and L.cl.tolist() == [2, 1]
    assert L.col.tolist() == [1, 0, 2, 3, 0, 1] and L.padding == 0


def test_spec_spmv_kats(port):
    n, uv, (row, col) = path4(port)
    L = port.build_slimsell(n, row, col, 2, 1)
    assert port.spmv_step(L, TROPICAL, np.array([0, KINF, KINF, KINF])).tolist() == [0, 1, KINF, KINF]
    assert port.spmv_step(L, SELMAX, np.array([1, 0, 0, 0])).tolist() == [1, 1, 0, 0]
    assert port.spmv_step(L, REAL, np.array([1, 1, 0, 1])).tolist() == [2, 2, 2, 1]


def test_spec_bfs_kats(port):
    n, uv, (row, col) = path4(port)
    L1 = port.build_slimsell(n, row, col, 2, 1)
    for v in (TROPICAL, REAL, BOOLEAN, SELMAX):
        out = port.bfs_spmv(L1, 0, v, csr=(row, col))
        assert out.dist.tolist() == [0, 1, 2, 3] and out.iterations == 4
        assert out.stats[:, 6].tolist() == [1, 1, 1, 0]
    L4 = port.build_slimsell(n, row, col, 2, 4)
    # the reference's sel-max root encoding
    assert port.bfs_spmv(L4, 0, SELMAX).parent.tolist() == [1, 1, 1, 2]
    assert port.bfs_spmv(L4, 2, SELMAX).parent.tolist() == [1, 0, 0, 0]


def test_reference_selftest_documents_quirk(golden):
    st = golden["ref_selftest"]
    assert st["exit"] == 2 and "selmax" in st["fail_lines"][0]


# ---- oracle vs the reference itself (container only) ------------------------

@pytest.mark.parametrize("scale,seed", [(6, 3), (9, 11)])
def test_port_matches_reference(port, ref, scale, seed):
    g = ref.gen_kronecker(scale, 8, seed)
    n, uv = port.gen_kronecker(scale, 8, seed)
    assert np.array_equal(uv, g.edges())
    row, col = port.to_csr(n, uv)
    for C_, sig in ((2, 1), (3, 5), (8, n), (32, n)):
        L = port.build_slimsell(n, row, col, C_, sig)
        r = ref.build_slimsell(g, C_, sig)
        Lr = r.layout()
        assert np.array_equal(L.col, Lr.col) and np.array_equal(L.perm, Lr.perm)
        for root in (0, n // 2, n - 1):
            for v in (TROPICAL, REAL, BOOLEAN, SELMAX):
                for sw, Lc in ((False, 0), (True, 4)):
                    a = port.bfs_spmv(L, root, v, sw, Lc, csr=(row, col))
                    b = ref.bfs_spmv(r, root, v, sw, Lc, csr_graph=g)
                    assert np.array_equal(a.dist, b.dist) and np.array_equal(a.parent, b.parent)
                    assert rows(a.stats) == rows(b.stats)


def test_port_edge_graphs_match_reference(port, ref, edge_graphs):
    """Pins the port on the edge cases the GPU suite replays on the device."""
    for name, n, uv in edge_graphs:
        g = ref.from_pairs(uv, n)
        assert np.array_equal(uv, g.edges()), name
        row, col = port.to_csr(n, uv)
        for C_, sig in ((1, 1), (8, n), (32, n), (32, 1)):
            L = port.build_slimsell(n, row, col, C_, sig)
            r = ref.build_slimsell(g, C_, sig)
            Lr = r.layout()
            assert np.array_equal(L.col, Lr.col) and np.array_equal(L.perm, Lr.perm), name
            for root in sorted({0, n // 2, n - 1}):
                for v in (TROPICAL, REAL, BOOLEAN, SELMAX):
                    for sw, Lc in ((False, 0), (True, 0), (True, 4)):
                        a = port.bfs_spmv(L, root, v, sw, Lc, csr=(row, col))
                        b = ref.bfs_spmv(r, root, v, sw, Lc, csr_graph=g)
                        key = (name, C_, sig, root, v, sw, Lc)
                        assert np.array_equal(a.dist, b.dist) and np.array_equal(a.parent, b.parent), key
                        assert rows(a.stats) == rows(b.stats), key


def test_port_er_matches_reference(port, ref):
    for n, p, seed in ((64, 0.15, 3), (500, 0.02, 9)):
        assert np.array_equal(port.gen_erdos_renyi(n, p, seed)[1], ref.gen_erdos_renyi(n, p, seed).edges())


def test_errors(port):
    n, uv, (row, col) = path4(port)
    from oracle import OracleError
    with pytest.raises(OracleError):
        port.build_slimsell(n, row, col, 0, 1)
    L = port.build_slimsell(n, row, col, 2, 1)
    with pytest.raises(OracleError):
        port.bfs_spmv(L, 4, TROPICAL)
    capped = port.bfs_spmv(L, 0, TROPICAL, max_iterations=2)
    assert capped.status == 3 and capped.dist.tolist()[:3] == [0, 1, 2]
