"""Host-side mirror of the reference's public API for the BFS-SpMV path.

Same names, argument meaning and error behaviour as
``/root/reference/proj/include/slimsell/{graph,generator,repr,semiring,bfs}.hpp``;
every call crosses the C-ABI of ``libslimsell_b200.so`` into sm_100a kernels.
Handles (``Graph``, ``SlimSellRepr``) are device-resident; arrays come back as
numpy int64 in the reference's layout.

Exception mapping (reference -> here): std::invalid_argument -> InvalidArgument
(a ValueError), std::out_of_range -> OutOfRange (an IndexError), BfsCapError ->
BfsCapError (carries ``partial``), CUDA failures -> DeviceError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib as _L

KINF = np.iinfo(np.int64).max  # semiring.hpp:20
NO_PARENT = -1                   # semiring.hpp:23
PAD_MARKER = -1                  # repr.hpp:14


class Variant(IntEnum):  # semiring.hpp:25
    tropical = 0
    real = 1
    boolean = 2
    selmax = 3


ALL_VARIANTS = (Variant.tropical, Variant.real, Variant.boolean, Variant.selmax)


class Schedule(IntEnum):  # bfs.hpp:14 (accepted; the device schedules itself)
    static_blocks = 0
    dynamic_queue = 1


class SlimSellError(RuntimeError):
    pass


class InvalidArgument(SlimSellError, ValueError):
    pass


class OutOfRange(SlimSellError, IndexError):
    pass


class DeviceError(SlimSellError):
    pass


class ParseError(SlimSellError):  # graph.hpp:15-21
    """Malformed input text; `line` is the 1-based line of the error."""

    def __init__(self, what: str):
        super().__init__(what)
        try:
            self.line = int(what.split(":", 1)[0].split()[1])
        except (IndexError, ValueError):
            self.line = 0


@dataclass
class IterStats:  # bfs.hpp:26-34
    iteration: int = 0
    elapsed_ns: int = 0
    chunks_processed: int = 0
    chunks_skipped: int = 0
    subchunks_processed: int = 0
    columns_processed: int = 0
    frontier_size: int = 0

    def counters(self):
        return (self.chunks_processed, self.chunks_skipped, self.subchunks_processed,
                self.columns_processed, self.frontier_size)


@dataclass
class BfsResult:  # bfs.hpp:36-42
    dist: np.ndarray
    parent: np.ndarray
    iterations: int
    per_iter: list = field(default_factory=list)

    @property
    def elapsed_ns(self) -> int:
        return sum(s.elapsed_ns for s in self.per_iter)


class BfsCapError(SlimSellError):  # bfs.hpp:46-54
    def __init__(self, what: str, partial: BfsResult):
        super().__init__(what)
        self.partial = partial


@dataclass
class BfsOptions:  # bfs.hpp:16-24 (+ selmax_compat)
    variant: Variant = Variant.tropical
    slimwork: bool = False
    slimchunk_len: int = 0
    schedule: Schedule = Schedule.static_blocks
    workers: int = 1
    max_iterations: int = 0
    want_parents: bool = True
    selmax_compat: bool = True

    def _c(self) -> _L.BfsOptionsC:
        return _L.BfsOptionsC(int(self.variant), int(bool(self.slimwork)), int(self.slimchunk_len),
                              int(self.schedule), int(self.workers), int(self.max_iterations),
                              int(bool(self.want_parents)), int(bool(self.selmax_compat)))


def _raise(rc: int):
    msg = _L.lib().ssb_last_error().decode(errors="replace")
    if rc == _L.SSB_EINVAL:
        raise InvalidArgument(msg)
    if rc == _L.SSB_ERANGE:
        raise OutOfRange(msg)
    if rc == _L.SSB_EPARSE:
        raise ParseError(msg)
    raise DeviceError(f"status {rc}: {msg}")


def _check(rc: int):
    if rc != _L.SSB_OK:
        _raise(rc)


def _p(a, ty=_L.i64p):
    return None if a is None else a.ctypes.data_as(ty)


def set_device(device: int) -> None:
    _check(_L.lib().ssb_set_device(device))


@dataclass
class CsrView:  # graph.hpp:63-69
    row: np.ndarray
    col: np.ndarray

    def num_vertices(self) -> int:
        return int(self.row.shape[0]) - 1


class Graph:
    """Normalised undirected graph, device-resident (graph.hpp:31-51)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        n, m = np.zeros(1, np.int64), np.zeros(1, np.int64)
        _check(_L.lib().ssb_edges_info(self._h, _p(n), _p(m)))
        self._n, self._m = int(n[0]), int(m[0])

    @staticmethod
    def from_pairs(pairs, n: int = -1) -> "Graph":  # graph.hpp:36
        uv = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
        h = C.c_void_p()
        _check(_L.lib().ssb_edges_from_pairs(_p(uv) if uv.size else None, uv.shape[0], n, C.byref(h)))
        return Graph(h)

    @staticmethod
    def from_edge_list(text, reject_asymmetric: bool = False) -> "Graph":  # graph.hpp:55
        t = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        _check(_L.lib().ssb_edges_from_edge_list(t, len(t), int(reject_asymmetric), C.byref(h)))
        return Graph(h)

    @staticmethod
    def from_matrix_market(text) -> "Graph":  # graph.hpp:59
        t = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        _check(_L.lib().ssb_edges_from_matrix_market(t, len(t), C.byref(h)))
        return Graph(h)

    def num_vertices(self) -> int:
        return self._n

    def num_edges(self) -> int:
        return self._m

    def edges(self) -> np.ndarray:
        uv = np.empty((self._m, 2), dtype=np.int64)
        if self._m:
            _check(_L.lib().ssb_edges_export(self._h, _p(uv)))
        return uv

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _L._lib is not None:
            _L._lib.ssb_edges_destroy(h)
            self._h = None


def _parsed(fn, *args):
    ptr, cnt, n = _L.i64p(), np.zeros(1, np.int64), np.zeros(1, np.int64)
    _check(fn(*args, C.byref(ptr), _p(cnt), _p(n)))
    try:
        k = int(cnt[0])
        uv = np.ctypeslib.as_array(ptr, shape=(max(2 * k, 1),))[: 2 * k].copy().reshape(-1, 2)
    finally:
        _L.lib().ssb_free(ptr)
    return int(n[0]), uv


def parse_edge_list(text, reject_asymmetric: bool = False):
    """The edge-list parser alone (host only): (declared n or -1, raw records)."""
    t = text.encode() if isinstance(text, str) else bytes(text)
    return _parsed(_L.lib().ssb_parse_edge_list, t, len(t), int(reject_asymmetric))


def parse_matrix_market(text):
    """The MatrixMarket parser alone (host only): (n, 0-based records)."""
    t = text.encode() if isinstance(text, str) else bytes(text)
    return _parsed(_L.lib().ssb_parse_matrix_market, t, len(t))


def gen_kronecker(scale: int, edgefactor: int, seed: int,
                  initiator=(0.57, 0.19, 0.19, 0.05)) -> Graph:  # generator.hpp:55
    h = C.c_void_p()
    _check(_L.lib().ssb_gen_kronecker(scale, edgefactor, seed, (C.c_double * 4)(*initiator), C.byref(h)))
    return Graph(h)


def gen_erdos_renyi(n: int, p: float, seed: int) -> Graph:  # generator.hpp:50
    h = C.c_void_p()
    _check(_L.lib().ssb_gen_erdos_renyi(n, p, seed, C.byref(h)))
    return Graph(h)


def gen_path(n: int) -> Graph:  # generator.hpp:62
    if n < 1:
        raise InvalidArgument("path needs n >= 1")
    return Graph.from_pairs(np.stack([np.arange(n - 1), np.arange(1, n)], 1), n)


def gen_clique(n: int) -> Graph:  # generator.hpp:63
    if n < 1:
        raise InvalidArgument("clique needs n >= 1")
    return Graph.from_pairs(np.stack(np.triu_indices(n, 1), 1), n)


def gen_star(n: int) -> Graph:  # generator.hpp:64
    if n < 1:
        raise InvalidArgument("star needs n >= 1")
    return Graph.from_pairs(np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1), n)


def to_csr(g: Graph) -> CsrView:  # graph.hpp:71
    row = np.empty(g.num_vertices() + 1, dtype=np.int64)
    col = np.empty(max(2 * g.num_edges(), 1), dtype=np.int64)
    _check(_L.lib().ssb_to_csr(g._h, _p(row), _p(col)))
    return CsrView(row, col[: 2 * g.num_edges()])


class SlimSellRepr:
    """Device-resident SlimSell layout (repr.hpp:33-55); arrays export lazily."""

    def __init__(self, handle):
        self._h = handle
        info = _L.LayoutInfo()
        _check(_L.lib().ssb_graph_info(self._h, C.byref(info)))
        self.C, self.sigma, self.n = info.C, info.sigma, info.n
        self.n_padded, self.n_chunks, self.nonzeros = info.n_padded, info.n_chunks, info.nonzeros
        self.n_cells, self.padding, self.max_chunk_len = info.n_cells, info.padding, info.max_chunk_len
        # cells held: chunks [range_begin, range_end) (the whole layout unless
        # built with build_slimsell(..., chunk_range=...))
        self.range_begin, self.range_end, self.range_cells = info.range_begin, info.range_end, info.range_cells
        self.range_segments = info.range_segments
        self._host = {}

    @property
    def partial(self) -> bool:
        return self.range_segments != 1 or self.range_begin > 0 or self.range_end < self.n_chunks

    def _export(self, name):
        if name not in self._host:
            if name in ("col", "cs"):
                col = np.empty(max(self.n_cells, 1), np.int64)
                cs = np.empty(max(self.n_chunks, 1), np.int64)
                _check(_L.lib().ssb_graph_export(self._h, _p(col), _p(cs), None, None, None))
                self._host.update(col=col[: self.n_cells], cs=cs[: self.n_chunks])
            elif name == "cl":
                cl = np.empty(max(self.n_chunks, 1), np.int64)
                _check(_L.lib().ssb_graph_export(self._h, None, None, _p(cl), None, None))
                self._host["cl"] = cl[: self.n_chunks]
            else:
                perm = np.empty(max(self.n, 1), np.int64)
                inv = np.empty(max(self.n, 1), np.int64)
                _check(_L.lib().ssb_graph_export(self._h, None, None, None, _p(perm), _p(inv)))
                self._host.update(perm=perm[: self.n], inv_perm=inv[: self.n])
        return self._host[name]

    col = property(lambda self: self._export("col"))
    cs = property(lambda self: self._export("cs"))
    cl = property(lambda self: self._export("cl"))
    perm = property(lambda self: self._export("perm"))
    inv_perm = property(lambda self: self._export("inv_perm"))

    def col32(self) -> np.ndarray:
        """The cells this handle holds (the whole col, or the range's)."""
        out = np.empty(max(self.range_cells, 1), np.int32)
        _check(_L.lib().ssb_graph_export_col32(self._h, _p(out, _L.i32p)))
        return out[: self.range_cells]

    def degrees(self) -> np.ndarray:
        """Degree of every original vertex id (row lengths of to_csr)."""
        out = np.empty(max(self.n, 1), np.int64)
        _check(_L.lib().ssb_graph_degrees(self._h, _p(out)))
        return out[: self.n]

    def chunk_row_begin(self, chunk: int) -> int:  # repr.hpp:47
        return chunk * self.C

    def chunk_row_end(self, chunk: int) -> int:  # repr.hpp:51-54
        return min((chunk + 1) * self.C, self.n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _L._lib is not None:
            _L._lib.ssb_graph_destroy(h)
            self._h = None


def build_slimsell(g: Graph, C_: int, sigma: int, chunk_range=None, segments=None) -> SlimSellRepr:  # repr.hpp:66
    """build_slimsell on the device. chunk_range=(b, e) or segments=[(b, e),
    ...]: one rank's share of a multi-GPU layout — the whole layout's perm /
    cl, the cells of those chunks only (ssb_build_slimsell_range/_segments)."""
    h = C.c_void_p()
    if segments is not None:
        b = np.array([x for seg in segments for x in seg], dtype=np.int64)
        _check(_L.lib().ssb_build_slimsell_segments(g._h, C_, sigma, _p(b), len(segments), C.byref(h)))
    elif chunk_range is None:
        _check(_L.lib().ssb_build_slimsell(g._h, C_, sigma, C.byref(h)))
    else:
        b, e = chunk_range
        _check(_L.lib().ssb_build_slimsell_range(g._h, C_, sigma, int(b), int(e), C.byref(h)))
    return SlimSellRepr(h)


def repr_from_layout(n, C_, sigma, nonzeros, col, cs, cl, perm) -> SlimSellRepr:
    """Upload a host SlimSellRepr's arrays (e.g. one built by the reference)."""
    col, cs, cl, perm = (np.ascontiguousarray(a, dtype=np.int64) for a in (col, cs, cl, perm))
    h = C.c_void_p()
    _check(_L.lib().ssb_graph_from_layout(n, C_, sigma, nonzeros, _p(col) if col.size else None,
                                          col.shape[0], _p(cs) if cs.size else None,
                                          _p(cl) if cl.size else None, cs.shape[0],
                                          _p(perm) if perm.size else None, C.byref(h)))
    return SlimSellRepr(h)


def spmv_step(r: SlimSellRepr, variant: Variant, x_prev, out=None, chunk_begin: int = 0,
              chunk_end: int | None = None) -> np.ndarray:  # repr.hpp:90-98
    x = np.ascontiguousarray(x_prev, dtype=np.int64)
    if x.shape[0] != r.n_padded:
        raise InvalidArgument(f"x_prev length {x.shape[0]}, expected {r.n_padded}")
    if out is None:
        out = np.zeros(r.n_padded, dtype=np.int64)
    elif out.shape[0] != r.n_padded or out.dtype != np.int64 or not out.flags.c_contiguous:
        raise InvalidArgument(f"out length {out.shape[0]}, expected {r.n_padded}")
    ce = r.n_chunks if chunk_end is None else chunk_end
    if r.n_padded == 0:
        return out
    _check(_L.lib().ssb_spmv_step(r._h, int(variant), _p(x), _p(out), chunk_begin, ce))
    return out


def spmv_step_device(r: SlimSellRepr, variant: Variant, x_prev, out, chunk_begin: int = 0,
                     chunk_end: int | None = None) -> float:
    """spmv_step with DEVICE operands (torch int64 CUDA tensors of n_padded):
    no host copies; returns the kernels' device time in ms."""
    for t, nm in ((x_prev, "x_prev"), (out, "out")):
        if not t.is_cuda or t.dtype.itemsize != 8 or t.numel() != r.n_padded or not t.is_contiguous():
            raise InvalidArgument(f"{nm} must be a contiguous int64 CUDA tensor of n_padded = {r.n_padded}")
    ce = r.n_chunks if chunk_end is None else chunk_end
    import torch
    torch.cuda.current_stream().synchronize()  # the library stream reads the tensors next
    ms = C.c_double()
    _check(_L.lib().ssb_spmv_step_device(r._h, int(variant), C.c_void_p(x_prev.data_ptr()),
                                         C.c_void_p(out.data_ptr()), chunk_begin, ce, C.byref(ms)))
    return float(ms.value)


def spmv_segment(r: SlimSellRepr, variant: Variant, x_prev, acc, chunk: int, col_begin: int,
                 col_len: int) -> np.ndarray:  # repr.hpp:79-81
    """acc[lane] = plus(acc[lane], times(x_prev[c], edge/pad)) over columns
    [col_begin, col_begin + col_len) of `chunk` (repr.cpp:20-35); acc is
    updated in place (C int64) and returned."""
    x = np.ascontiguousarray(x_prev, dtype=np.int64)
    if x.shape[0] != r.n_padded:
        raise InvalidArgument(f"x_prev length {x.shape[0]}, expected {r.n_padded}")
    if acc.shape[0] != r.C or acc.dtype != np.int64 or not acc.flags.c_contiguous:
        raise InvalidArgument(f"acc must be contiguous int64[C = {r.C}]")
    _check(_L.lib().ssb_spmv_segment(r._h, int(variant), _p(x), _p(acc), chunk, col_begin, col_len))
    return acc


def _stats_list(buf, k):
    return [IterStats(s.iteration, s.elapsed_ns, s.chunks_processed, s.chunks_skipped,
                      s.subchunks_processed, s.columns_processed, s.frontier_size) for s in buf[:k]]


def bfs_spmv(r: SlimSellRepr, root: int, opts: BfsOptions | None = None,
             csr_for_parents: CsrView | None = None, out_dist: np.ndarray | None = None,
             out_parent: np.ndarray | None = None) -> BfsResult:  # bfs.hpp:80-81
    """Algebraic BFS on the device. As the reference: sel-max always produces
    parents when opts.want_parents; the other variants only when a CSR is
    passed (they are derived from the distances, dp_transform semantics).
    out_dist / out_parent may be caller-owned (e.g. pinned) int64[n] buffers;
    the result then aliases them instead of copying."""
    opts = opts or BfsOptions()
    want = bool(opts.want_parents) and (opts.variant == Variant.selmax or csr_for_parents is not None)
    o = opts._c()
    o.want_parents = int(want)
    n = r.n
    for buf in (out_dist, out_parent):
        if buf is not None and (buf.dtype != np.int64 or buf.shape[0] < n or not buf.flags.c_contiguous):
            raise InvalidArgument("output buffers must be contiguous int64[n]")
    dist = np.empty(max(n, 1), np.int64) if out_dist is None else out_dist
    parent = np.empty(max(n, 1), np.int64) if out_parent is None else out_parent
    plen = np.zeros(1, np.int64)
    iters = np.zeros(1, np.int64)
    cap = min(max(n + 2, 2), 1 << 12)  # deeper BFS: rerun below with an exact-size buffer
    while True:
        stats = (_L.IterStatsC * cap)()
        rc = _L.lib().ssb_bfs_spmv(r._h, int(root), C.byref(o), _p(dist), _p(parent), _p(plen),
                                   stats, cap, _p(iters))
        if rc not in (_L.SSB_OK, _L.SSB_ECAP):
            _raise(rc)
        k = int(iters[0])
        if k <= cap:
            break
        cap = k  # deeper than the first buffer: rerun once with room for every record
    keep = (lambda a: a[:n]) if out_dist is not None else (lambda a: a[:n].copy())
    res = BfsResult(keep(dist), parent[: int(plen[0])] if out_parent is not None else
                    parent[: int(plen[0])].copy(), k, _stats_list(stats, k))
    if rc == _L.SSB_ECAP:
        raise BfsCapError(_L.lib().ssb_last_error().decode(), res)
    return res


def bfs_spmv_batch(r: SlimSellRepr, roots, opts: BfsOptions | None = None,
                   csr_for_parents: CsrView | None = None, out_dists=None, out_parents=None):
    """A Graph500 root list through ssb_bfs_spmv_batch: root i's result lands in
    out_dists[i] / out_parents[i] (contiguous int64[n]; entries may repeat — a
    later root's result then replaces an earlier one's) while the next root's
    BFS runs on the device. Parents as bfs_spmv (sel-max, or any variant with
    a CSR). Returns the per-root iteration counts; BfsCapError carries the
    capped root's index as .root_index."""
    opts = opts or BfsOptions()
    roots = np.ascontiguousarray(roots, dtype=np.int64)
    k = roots.shape[0]
    n = r.n
    want = bool(opts.want_parents) and (opts.variant == Variant.selmax or csr_for_parents is not None)
    o = opts._c()
    o.want_parents = int(want)
    if out_dists is None:
        out_dists = [np.empty(max(n, 1), np.int64) for _ in range(k)]
    if want and out_parents is None:
        out_parents = [np.empty(max(n, 1), np.int64) for _ in range(k)]
    for buf in list(out_dists) + list(out_parents or []):
        if buf.dtype != np.int64 or buf.shape[0] < n or not buf.flags.c_contiguous:
            raise InvalidArgument("output buffers must be contiguous int64[n]")
    dp = (_L.i64p * max(k, 1))(*[_p(out_dists[i]) for i in range(k)])
    pp = (_L.i64p * max(k, 1))(*[_p(out_parents[i]) for i in range(k)]) if want else None
    iters = np.zeros(max(k, 1), np.int64)
    capped = np.zeros(1, np.int64)
    rc = _L.lib().ssb_bfs_spmv_batch(r._h, _p(roots), k, C.byref(o), dp, pp, _p(iters), _p(capped))
    if rc == _L.SSB_ECAP:
        i = int(capped[0])
        e = BfsCapError(_L.lib().ssb_last_error().decode(),
                        BfsResult(out_dists[i][:n], np.empty(0, np.int64), int(iters[i]), []))
        e.root_index = i
        raise e
    _check(rc)
    return [int(x) for x in iters[:k]]


def bfs_traditional(g: Graph, root: int) -> BfsResult:  # bfs.hpp:86, bfs.cpp:248-291
    """The reference's queue BFS, on the device over the graph's CSR: parent =
    smallest neighbour one level closer, root self-parented."""
    n = g.num_vertices()
    dist = np.empty(max(n, 1), np.int64)
    parent = np.empty(max(n, 1), np.int64)
    cap = min(n + 2, 4096)
    st = (_L.IterStatsC * cap)()
    it = np.zeros(1, np.int64)
    _check(_L.lib().ssb_bfs_traditional(g._h, root, _p(dist), _p(parent), st, cap, _p(it)))
    k = int(it[0])
    if k > cap:
        st = (_L.IterStatsC * k)()
        _check(_L.lib().ssb_bfs_traditional(g._h, root, _p(dist), _p(parent), st, k, _p(it)))
    per = [IterStats(iteration=s.iteration, elapsed_ns=s.elapsed_ns, frontier_size=s.frontier_size)
           for s in st[:k]]
    return BfsResult(dist[:n], parent[:n], k, per)


VALIDATE_SELMAX_COMPAT, VALIDATE_MIN_PARENT_EXACT, VALIDATE_SELMAX_EXACT = 1, 2, 4


def validate_bfs(g: Graph, root: int, dist, parent=None, selmax_compat: bool = False,
                 exact: str | None = None, layout: "SlimSellRepr | None" = None):
    """cli.cpp:73-112 (the parent-tree checks of verify_against_oracle) plus the
    Graph500 edge checks, on the device. Returns None when valid, else a report
    (the first few violations) — the reference's optional<string>.

    exact="min": every parent must be the smallest original-id neighbour one
    level closer (dp_transform / bfs_traditional; tropical, real, boolean).
    exact="selmax": every parent must be the reference's sel-max value
    perm[max position of a neighbour one level closer], with the root encoding
    (perm[root] at levels 0-1) when selmax_compat; needs
    the layout the BFS ran on. Together with the edge checks this pins dist
    and parent bit for bit at any scale."""
    dist = np.ascontiguousarray(dist, dtype=np.int64)
    par = None if parent is None or len(parent) == 0 else np.ascontiguousarray(parent, dtype=np.int64)
    if dist.shape[0] != g.num_vertices() or (par is not None and par.shape[0] != g.num_vertices()):
        raise InvalidArgument("dist/parent length must equal the vertex count")
    flags = VALIDATE_SELMAX_COMPAT if selmax_compat else 0
    if exact == "min":
        flags |= VALIDATE_MIN_PARENT_EXACT
    elif exact == "selmax":
        flags |= VALIDATE_SELMAX_EXACT
    elif exact is not None:
        raise InvalidArgument("exact must be None, 'min' or 'selmax'")
    bad = np.zeros(1, np.int64)
    buf = C.create_string_buffer(1024)
    _check(_L.lib().ssb_validate_bfs_exact(g._h, layout._h if layout is not None else None, root, _p(dist),
                                           _p(par), flags, _p(bad), buf, 1024))
    if int(bad[0]) == 0:
        return None
    return f"{int(bad[0])} violation(s):\n" + buf.value.decode()


class DeviceBfs:
    """Benchmark-facing form: BFS results stay on the device (ssb_bfs_run)."""

    def __init__(self, r: SlimSellRepr):
        self.r = r
        self._stats = (_L.IterStatsC * 4096)()

    def run(self, root: int, opts: BfsOptions):
        it = np.zeros(1, np.int64)
        ms = C.c_double()
        o = opts._c()
        rc = _L.lib().ssb_bfs_run(self.r._h, int(root), C.byref(o), self._stats, 4096, _p(it), C.byref(ms))
        if rc not in (_L.SSB_OK, _L.SSB_ECAP):
            _raise(rc)
        k = int(it[0])
        return k, float(ms.value), _stats_list(self._stats, min(k, 4096)), rc

    def fetch(self, want_parents: bool, dist=None, parent=None):
        n = self.r.n
        dist = np.empty(n, np.int64) if dist is None else dist
        parent = np.empty(n, np.int64) if parent is None else parent
        plen = np.zeros(1, np.int64)
        _check(_L.lib().ssb_bfs_fetch(self.r._h, int(want_parents), _p(dist), _p(parent), _p(plen)))
        return dist, parent[: int(plen[0])]

    def last_timing(self):
        """(kernel_ms, launches) of the last run."""
        ms = C.c_double()
        n = np.zeros(1, np.int64)
        _check(_L.lib().ssb_bfs_last_timing(self.r._h, C.byref(ms), _p(n)))
        return float(ms.value), int(n[0])

    def edges_traversed(self) -> int:
        m = np.zeros(1, np.int64)
        _check(_L.lib().ssb_bfs_edges_traversed(self.r._h, _p(m)))
        return int(m[0])

    def columns_swept(self) -> int:
        """Columns the last run streamed (<= Σ columns_processed: early exit)."""
        m = np.zeros(1, np.int64)
        _check(_L.lib().ssb_bfs_columns_swept(self.r._h, _p(m)))
        return int(m[0])
