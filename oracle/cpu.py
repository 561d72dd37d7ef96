"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

See ``oracle/__init__.py`` for who may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libslimsell_ref.so")
REF_DIR = os.environ.get("SLIMSELL_REF_DIR", "/root/reference/proj")

KINF = np.iinfo(np.int64).max
TROPICAL, REAL, BOOLEAN, SELMAX = 0, 1, 2, 3
VARIANTS = {"tropical": TROPICAL, "real": REAL, "boolean": BOOLEAN, "selmax": SELMAX}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def build(ref: bool = True, alongside: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present; with
    ``alongside`` also _ref/test_alongside, which links libslimsell_b200.so)."""
    targets = ["liboracle.so"]
    if ref and os.path.isdir(REF_DIR):
        targets.append("ref")
        if alongside:
            targets.append("alongside")
    subprocess.run(["make", "-s", "-C", HERE, f"REF={REF_DIR}", *targets], check=True)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def _p(a: np.ndarray | None, ty=_i64p):
    if a is None:
        return None
    return a.ctypes.data_as(ty)


@dataclass
class Layout:
    """A SlimSellRepr as plain int64 arrays (repr.hpp:33-55)."""

    C: int
    sigma: int
    n: int
    n_padded: int
    n_chunks: int
    nonzeros: int
    padding: int
    col: np.ndarray
    cs: np.ndarray
    cl: np.ndarray
    perm: np.ndarray
    inv_perm: np.ndarray

    @property
    def n_cells(self) -> int:
        return int(self.col.shape[0])


@dataclass
class BfsOut:
    dist: np.ndarray
    parent: np.ndarray  # empty when not produced
    iterations: int
    stats: np.ndarray  # (iterations, 7): iteration, elapsed_ns, chunks_processed,
    # chunks_skipped, subchunks_processed, columns_processed, frontier_size
    status: int = 0


class _SoRepr(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("C", "sigma", "n", "n_padded", "n_chunks", "nonzeros", "n_cells", "padding")] + \
               [(k, _i64p) for k in ("col", "cs", "cl", "perm", "inv_perm")]


class Port:
    """The plain-C restatement (liboracle.so)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.so_gen_kronecker_pairs.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_double), _i64p]
        L.so_gen_erdos_renyi_pairs.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.POINTER(_i64p), _i64p]
        L.so_normalize_pairs.argtypes = [_i64p, C.c_int64, C.c_int64, _i64p]
        L.so_normalize_pairs.restype = C.c_int64
        L.so_to_csr.argtypes = [C.c_int64, _i64p, C.c_int64, _i64p, _i64p]
        L.so_build_slimsell.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, C.c_int64, C.POINTER(_SoRepr)]
        L.so_repr_free.argtypes = [C.POINTER(_SoRepr)]
        L.so_spmv_step.argtypes = [C.POINTER(_SoRepr), C.c_int, _i64p, _i64p, C.c_int64, C.c_int64]
        L.so_bfs_spmv.argtypes = [C.POINTER(_SoRepr), C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                  C.c_int, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, C.c_int64]
        L.so_bfs_traditional.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, _i64p, _i64p, _i64p]
        L.so_dp_transform.argtypes = [C.c_int64, _i64p, _i64p, _i64p, _i64p]
        L.so_pick_roots.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _i64p]
        L.so_mix64.argtypes = [C.c_uint64]
        L.so_mix64.restype = C.c_uint64
        L.so_fnv1a64.argtypes = [C.c_void_p, C.c_int64]
        L.so_fnv1a64.restype = C.c_uint64
        L.so_fnv1a64_i32.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        L.so_fnv1a64_i32.restype = C.c_uint64

    # -- generators / graph core ------------------------------------------
    def gen_kronecker_pairs(self, scale, ef, seed, init=(0.57, 0.19, 0.19, 0.05)):
        uv = np.empty(2 * (ef << scale), dtype=np.int64)
        a = (C.c_double * 4)(*init)
        rc = self.lib.so_gen_kronecker_pairs(scale, ef, seed, a, _p(uv))
        if rc:
            raise OracleError(rc)
        return uv.reshape(-1, 2)

    def from_pairs(self, pairs, n=-1):
        uv = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2).copy()
        n_out = np.zeros(1, dtype=np.int64)
        m = self.lib.so_normalize_pairs(_p(uv), uv.shape[0], n, _p(n_out))
        if m < 0:
            raise OracleError(-m, "vertex id out of range")
        return int(n_out[0]), uv[:m].copy()

    def gen_kronecker(self, scale, ef, seed, init=(0.57, 0.19, 0.19, 0.05)):
        return self.from_pairs(self.gen_kronecker_pairs(scale, ef, seed, init), 1 << scale)

    def gen_erdos_renyi(self, n, p, seed):
        ptr = _i64p()
        cnt = C.c_int64()
        rc = self.lib.so_gen_erdos_renyi_pairs(n, p, seed, C.byref(ptr), C.byref(cnt))
        if rc:
            raise OracleError(rc)
        pairs = np.ctypeslib.as_array(ptr, shape=(max(cnt.value, 1) * 2,))[: 2 * cnt.value].copy()
        C.CDLL(None).free(ptr)
        return self.from_pairs(pairs.reshape(-1, 2), n)

    @staticmethod
    def gen_path(n):
        return n, np.stack([np.arange(n - 1), np.arange(1, n)], 1).astype(np.int64)

    @staticmethod
    def gen_clique(n):
        iu = np.triu_indices(n, 1)
        return n, np.stack(iu, 1).astype(np.int64)

    @staticmethod
    def gen_star(n):
        return n, np.stack([np.zeros(n - 1), np.arange(1, n)], 1).astype(np.int64)

    def to_csr(self, n, uv):
        uv = np.ascontiguousarray(uv, dtype=np.int64)
        row = np.empty(n + 1, dtype=np.int64)
        col = np.empty(2 * uv.shape[0], dtype=np.int64)
        self.lib.so_to_csr(n, _p(uv), uv.shape[0], _p(row), _p(col))
        return row, col

    # -- layout --------------------------------------------------------------
    def build_slimsell(self, n, row, col, Cc, sigma) -> Layout:
        s = _SoRepr()
        rc = self.lib.so_build_slimsell(n, _p(row), _p(col), Cc, sigma, C.byref(s))
        if rc:
            raise OracleError(rc)
        cp = lambda ptr, k: np.ctypeslib.as_array(ptr, shape=(max(k, 1),))[:k].copy()  # noqa: E731
        out = Layout(s.C, s.sigma, s.n, s.n_padded, s.n_chunks, s.nonzeros, s.padding,
                     cp(s.col, s.n_cells), cp(s.cs, s.n_chunks), cp(s.cl, s.n_chunks),
                     cp(s.perm, s.n), cp(s.inv_perm, s.n))
        self.lib.so_repr_free(C.byref(s))
        return out

    @staticmethod
    def _so(L: Layout) -> _SoRepr:
        s = _SoRepr(L.C, L.sigma, L.n, L.n_padded, L.n_chunks, L.nonzeros, L.n_cells, L.padding)
        L._keep = [np.ascontiguousarray(a, dtype=np.int64) for a in (L.col, L.cs, L.cl, L.perm, L.inv_perm)]
        s.col, s.cs, s.cl, s.perm, s.inv_perm = (_p(a) for a in L._keep)
        return s

    def spmv_step(self, L: Layout, variant, x_prev, out=None, chunk_begin=0, chunk_end=None):
        x = np.ascontiguousarray(x_prev, dtype=np.int64)
        out = np.zeros(L.n_padded, dtype=np.int64) if out is None else out
        ce = L.n_chunks if chunk_end is None else chunk_end
        rc = self.lib.so_spmv_step(C.byref(self._so(L)), variant, _p(x), _p(out), chunk_begin, ce)
        if rc:
            raise OracleError(rc)
        return out

    def bfs_spmv(self, L: Layout, root, variant, slimwork=False, slimchunk_len=0,
                 max_iterations=0, want_parents=True, csr=None) -> BfsOut:
        dist = np.empty(max(L.n, 1), dtype=np.int64)
        parent = np.empty(max(L.n, 1), dtype=np.int64)
        plen = np.zeros(1, dtype=np.int64)
        iters = np.zeros(1, dtype=np.int64)
        cap = L.n + 2
        stats = np.zeros((cap, 7), dtype=np.int64)
        row, col = (None, None) if csr is None else csr
        rc = self.lib.so_bfs_spmv(C.byref(self._so(L)), root, variant, int(slimwork), slimchunk_len,
                                  max_iterations, int(want_parents), _p(row), _p(col), _p(dist),
                                  _p(parent), _p(plen), _p(iters), _p(stats), cap)
        if rc not in (0, 3):
            raise OracleError(rc)
        k = int(iters[0])
        return BfsOut(dist[: L.n], parent[: int(plen[0])], k, stats[:k], rc)

    def bfs_traditional(self, n, row, col, root):
        dist = np.empty(n, dtype=np.int64)
        parent = np.empty(n, dtype=np.int64)
        it = np.zeros(1, dtype=np.int64)
        rc = self.lib.so_bfs_traditional(n, _p(row), _p(col), root, _p(dist), _p(parent), _p(it))
        if rc:
            raise OracleError(rc)
        return dist, parent, int(it[0])

    def dp_transform(self, n, row, col, d):
        parent = np.empty(n, dtype=np.int64)
        d = np.ascontiguousarray(d, dtype=np.int64)
        rc = self.lib.so_dp_transform(n, _p(row), _p(col), _p(d), _p(parent))
        if rc:
            raise OracleError(rc)
        return parent

    def pick_roots(self, n, want, seed):
        want = min(max(want, 1), n)
        roots = np.empty(want, dtype=np.int64)
        self.lib.so_pick_roots(n, want, seed, _p(roots))
        return roots

    def mix64(self, x):
        return self.lib.so_mix64(x)

    def fnv_i32(self, a) -> str:
        """fnv() of an int32 array's values as int64 (no widened copy)."""
        a = np.ascontiguousarray(a, dtype=np.int32)
        return format(self.lib.so_fnv1a64_i32(a.ctypes.data, a.shape[0], 0xCBF29CE484222325), "016x")

    def fnv(self, a) -> str:
        """FNV-1a-64 of an array's little-endian int64 bytes, as 16 hex digits."""
        a = np.ascontiguousarray(a, dtype=np.int64)
        return format(self.lib.so_fnv1a64(a.ctypes.data, a.nbytes), "016x")


class RefGraph:
    def __init__(self, ref: "Reference", h):
        self.ref, self.h = ref, h

    @property
    def n(self):
        return self.ref.lib.ref_graph_n(self.h)

    @property
    def m(self):
        return self.ref.lib.ref_graph_m(self.h)

    def edges(self):
        uv = np.empty((self.m, 2), dtype=np.int64)
        self.ref.lib.ref_graph_edges(self.h, _p(uv))
        return uv

    def edges_fnv(self) -> str:
        return format(self.ref.lib.ref_graph_edges_fnv(self.h), "016x")

    def degrees(self) -> np.ndarray:
        deg = np.empty(self.n, dtype=np.int64)
        self.ref.lib.ref_graph_degrees(self.h, _p(deg))
        return deg

    def drop_csr(self):
        self.ref.lib.ref_graph_drop_csr(self.h)

    def csr(self):
        row = np.empty(self.n + 1, dtype=np.int64)
        col = np.empty(2 * self.m, dtype=np.int64)
        self.ref.lib.ref_graph_csr(self.h, _p(row), _p(col))
        return row, col

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass


class RefRepr:
    def __init__(self, ref: "Reference", h):
        self.ref, self.h = ref, h
        info = np.zeros(8, dtype=np.int64)
        ref.lib.ref_repr_info(h, _p(info))
        (self.C, self.sigma, self.n, self.n_padded, self.n_chunks, self.nonzeros,
         self.n_cells, self.padding) = (int(v) for v in info)

    def fnv(self, which: str) -> str:
        """In-place FNV-1a-64 of col / cs / cl / perm / inv_perm."""
        k = ("col", "cs", "cl", "perm", "inv_perm").index(which)
        return format(self.ref.lib.ref_repr_fnv(self.h, k), "016x")

    def layout(self) -> Layout:
        col = np.empty(self.n_cells, dtype=np.int64)
        cs = np.empty(self.n_chunks, dtype=np.int64)
        cl = np.empty(self.n_chunks, dtype=np.int64)
        perm = np.empty(self.n, dtype=np.int64)
        inv = np.empty(self.n, dtype=np.int64)
        self.ref.lib.ref_repr_export(self.h, _p(col), _p(cs), _p(cl), _p(perm), _p(inv))
        return Layout(self.C, self.sigma, self.n, self.n_padded, self.n_chunks, self.nonzeros,
                      self.padding, col, cs, cl, perm, inv)

    def __del__(self):
        try:
            self.ref.lib.ref_repr_free(self.h)
        except Exception:
            pass


class Reference:
    """The unmodified reference library through the C shim (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen_kronecker.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_double), C.POINTER(vp)]
        L.ref_gen_erdos_renyi.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.POINTER(vp)]
        L.ref_gen_named.argtypes = [C.c_int, C.c_int64, C.POINTER(vp)]
        L.ref_graph_from_pairs.argtypes = [_i64p, C.c_int64, C.c_int64, C.POINTER(vp)]
        L.ref_from_edge_list.argtypes = [C.c_char_p, C.c_int64, C.c_int, C.POINTER(vp)]
        L.ref_from_matrix_market.argtypes = [C.c_char_p, C.c_int64, C.POINTER(vp)]
        L.ref_graph_n.argtypes = [vp]
        L.ref_graph_n.restype = C.c_int64
        L.ref_graph_m.argtypes = [vp]
        L.ref_graph_m.restype = C.c_int64
        L.ref_graph_edges.argtypes = [vp, _i64p]
        L.ref_graph_csr.argtypes = [vp, _i64p, _i64p]
        L.ref_graph_free.argtypes = [vp]
        L.ref_build_slimsell.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(vp)]
        L.ref_repr_from_arrays.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i32p, C.c_int64,
                                           _i64p, _i64p, C.c_int64, _i64p, _i64p, C.POINTER(vp)]
        L.ref_repr_info.argtypes = [vp, _i64p]
        L.ref_repr_export.argtypes = [vp, _i64p, _i64p, _i64p, _i64p, _i64p]
        L.ref_repr_free.argtypes = [vp]
        L.ref_spmv_step.argtypes = [vp, C.c_int, _i64p, _i64p, C.c_int64, C.c_int64]
        L.ref_permute_in.argtypes = [vp, _i64p, C.c_int64, _i64p]
        L.ref_permute_out.argtypes = [vp, _i64p, _i64p]
        L.ref_bfs_spmv.argtypes = [vp, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int64,
                                   C.c_int, vp, _i64p, _i64p, _i64p, _i64p, _i64p, C.c_int64]
        L.ref_bfs_traditional.argtypes = [vp, C.c_int64, _i64p, _i64p, _i64p]
        L.ref_dp_transform.argtypes = [vp, _i64p, _i64p]
        L.ref_selftest.argtypes = [C.c_uint64, C.c_int, C.c_char_p, C.c_int64]
        L.ref_graph_edges_fnv.argtypes = [vp]
        L.ref_graph_edges_fnv.restype = C.c_uint64
        L.ref_graph_degrees.argtypes = [vp, _i64p]
        L.ref_graph_drop_csr.argtypes = [vp]
        L.ref_repr_fnv.argtypes = [vp, C.c_int]
        L.ref_repr_fnv.restype = C.c_uint64
        L.ref_bfs_traditional_timed.argtypes = [vp, C.c_int64, _i64p, _i64p, _i64p, _i64p]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _graph(self, fn, *args) -> RefGraph:
        h = C.c_void_p()
        self._check(fn(*args, C.byref(h)))
        return RefGraph(self, h)

    def gen_kronecker(self, scale, ef, seed, init=(0.57, 0.19, 0.19, 0.05)) -> RefGraph:
        return self._graph(self.lib.ref_gen_kronecker, scale, ef, seed, (C.c_double * 4)(*init))

    def gen_erdos_renyi(self, n, p, seed) -> RefGraph:
        return self._graph(self.lib.ref_gen_erdos_renyi, n, p, seed)

    def gen_path(self, n):
        return self._graph(self.lib.ref_gen_named, 0, n)

    def gen_clique(self, n):
        return self._graph(self.lib.ref_gen_named, 1, n)

    def gen_star(self, n):
        return self._graph(self.lib.ref_gen_named, 2, n)

    def from_pairs(self, pairs, n=-1) -> RefGraph:
        uv = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
        return self._graph(self.lib.ref_graph_from_pairs, _p(uv), uv.shape[0], n)

    def from_edge_list(self, text: bytes, reject_asymmetric=False) -> RefGraph:
        return self._graph(self.lib.ref_from_edge_list, text, len(text), int(reject_asymmetric))

    def from_matrix_market(self, text: bytes) -> RefGraph:
        return self._graph(self.lib.ref_from_matrix_market, text, len(text))

    def build_slimsell(self, g: RefGraph, Cc, sigma) -> RefRepr:
        h = C.c_void_p()
        self._check(self.lib.ref_build_slimsell(g.h, Cc, sigma, C.byref(h)))
        return RefRepr(self, h)

    def repr_from_arrays(self, n, Cc, sigma, nonzeros, col32, cs, cl, perm, inv_perm) -> RefRepr:
        h = C.c_void_p()
        col32 = np.ascontiguousarray(col32, dtype=np.int32)
        cs, cl, perm, inv_perm = (np.ascontiguousarray(a, dtype=np.int64) for a in (cs, cl, perm, inv_perm))
        self._check(self.lib.ref_repr_from_arrays(n, Cc, sigma, nonzeros, _p(col32, _i32p), col32.shape[0],
                                                  _p(cs), _p(cl), cs.shape[0], _p(perm), _p(inv_perm),
                                                  C.byref(h)))
        return RefRepr(self, h)

    def spmv_step(self, r: RefRepr, variant, x_prev, out=None, chunk_begin=0, chunk_end=None):
        x = np.ascontiguousarray(x_prev, dtype=np.int64)
        out = np.zeros(r.n_padded, dtype=np.int64) if out is None else out
        ce = r.n_chunks if chunk_end is None else chunk_end
        self._check(self.lib.ref_spmv_step(r.h, variant, _p(x), _p(out), chunk_begin, ce))
        return out

    def bfs_spmv(self, r: RefRepr, root, variant, slimwork=False, slimchunk_len=0, schedule=1,
                 workers=1, max_iterations=0, want_parents=True, csr_graph: RefGraph | None = None) -> BfsOut:
        n = r.n
        dist = np.empty(max(n, 1), dtype=np.int64)
        parent = np.empty(max(n, 1), dtype=np.int64)
        plen = np.zeros(1, dtype=np.int64)
        iters = np.zeros(1, dtype=np.int64)
        cap = n + 2
        stats = np.zeros((cap, 7), dtype=np.int64)
        rc = self.lib.ref_bfs_spmv(r.h, root, variant, int(slimwork), slimchunk_len, schedule, workers,
                                   max_iterations, int(want_parents), csr_graph.h if csr_graph else None,
                                   _p(dist), _p(parent), _p(plen), _p(iters), _p(stats), cap)
        if rc not in (0, 3):
            self._check(rc)
        k = int(iters[0])
        return BfsOut(dist[:n], parent[: int(plen[0])], k, stats[:k], rc)

    def bfs_traditional(self, g: RefGraph, root):
        n = g.n
        dist = np.empty(n, dtype=np.int64)
        parent = np.empty(n, dtype=np.int64)
        it = np.zeros(1, dtype=np.int64)
        self._check(self.lib.ref_bfs_traditional(g.h, root, _p(dist), _p(parent), _p(it)))
        return dist, parent, int(it[0])

    def bfs_traditional_timed(self, g: RefGraph, root, want=True):
        """bfs_traditional plus Σ IterStats.elapsed_ns (seconds)."""
        n = g.n
        dist = np.empty(n, dtype=np.int64) if want else None
        parent = np.empty(n, dtype=np.int64) if want else None
        it = np.zeros(1, dtype=np.int64)
        ns = np.zeros(1, dtype=np.int64)
        self._check(self.lib.ref_bfs_traditional_timed(g.h, root, _p(dist), _p(parent), _p(it), _p(ns)))
        return dist, parent, int(it[0]), float(ns[0]) * 1e-9

    def dp_transform(self, g: RefGraph, d):
        parent = np.empty(g.n, dtype=np.int64)
        d = np.ascontiguousarray(d, dtype=np.int64)
        self._check(self.lib.ref_dp_transform(g.h, _p(d), _p(parent)))
        return parent

    def selftest(self, seed=7, workers=8):
        buf = C.create_string_buffer(1 << 16)
        rc = self.lib.ref_selftest(seed, workers, buf, len(buf))
        return rc, buf.value.decode(errors="replace")
