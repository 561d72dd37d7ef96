"""Host-side plumbing of the multi-GPU BFS-SpMV.

Two decompositions:

* ``root_shard`` — root-parallel (the S26 bench): every rank holds the whole
  graph and runs roots[rank::world]; no data-path collective.
* chunk-range sharding (the S28 design): ranks own contiguous, cell-balanced
  chunk ranges and the replicated 1-bit frontier. Each BFS iteration ends with
  ONE exchange: every rank contributes the frontier words of its chunk range
  (C = 32 ⇒ chunk i ↔ word i), all ranks all-gather them, and "no row newly
  reached anywhere" — the reference's is_converged (semiring.cpp:152-157) — is
  read off the gathered words, so no extra all-reduce is needed. Counters are
  summed once at the end.

``ShardedFrontierExchange`` is the collective step, written against
``torch.distributed`` (NCCL on B200s, gloo in the CPU tests). The per-rank
sweep is supplied by the caller (the device kernel in the product; a plain
numpy sweep in tests/test_multirank.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def root_shard(roots, rank: int, world: int):
    """Roots a rank runs in the root-parallel decomposition."""
    return list(roots)[rank::world]


def partition_chunks(cl: np.ndarray, C: int, world: int) -> list[tuple[int, int]]:
    """Contiguous chunk ranges [b, e) with near-equal cell counts (C·cl) and at
    least one chunk each while chunks remain (SURVEY.md §8(e) "contiguous,
    cell-balanced")."""
    cl = np.asarray(cl, dtype=np.int64)
    nc = cl.shape[0]
    if world < 1:
        raise ValueError("world must be >= 1")
    # +1 per chunk so cell-less chunks still spread (their visited words count)
    w = C * cl + 1
    cum = np.concatenate([[0], np.cumsum(w)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r // world
        b = int(np.searchsorted(cum, target, side="left"))
        b = min(max(b, bounds[-1]), nc)
        bounds.append(b)
    bounds.append(nc)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def partition_segments(cl: np.ndarray, C: int, world: int, k: int) -> list[list[tuple[int, int]]]:
    """k·world contiguous cell-balanced pieces dealt to the ranks in snake
    order (0..W-1, W-1..0, ...): every rank gets k segments spread over the
    whole id range, so the hub chunks at the front — skipped once SlimWork
    marks them visited — do not idle one rank ("deal
    cell-balanced segments round-robin"). k = 1 is partition_chunks."""
    if k < 1:
        raise ValueError("k must be >= 1")
    pieces = partition_chunks(cl, C, world * k)
    out: list[list[tuple[int, int]]] = [[] for _ in range(world)]
    for j, pc in enumerate(pieces):
        rnd, pos = divmod(j, world)
        out[pos if rnd % 2 == 0 else world - 1 - pos].append(pc)
    return out


def _segments_of(spec) -> list[tuple[int, int]]:
    """(b, e) or [(b, e), ...] -> [(b, e), ...]"""
    if len(spec) == 2 and all(isinstance(x, (int, np.integer)) for x in spec):
        return [(int(spec[0]), int(spec[1]))]
    return [(int(b), int(e)) for b, e in spec]


@dataclass
class ExchangeResult:
    frontier: np.ndarray  # full frontier bitmap words (uint32)
    any_new: bool
    newly: int


class ShardedFrontierExchange:
    """All-gather of per-rank frontier word ranges into the replicated bitmap.

    Slices are padded to the longest range so one ``all_gather_into_tensor``
    suffices; with C = 32 a chunk range [b, e) is exactly word range [b, e).
    """

    def __init__(self, ranges: list[tuple[int, int]], n_words: int, dist, group=None, device="cpu"):
        import torch

        self.ranges = ranges
        self.n_words = n_words
        self.dist = dist
        self.group = group
        self.world = len(ranges)
        self.slot = max(1, max(e - b for b, e in ranges))
        self.device = device
        self._send = torch.zeros(self.slot, dtype=torch.int32, device=device)
        self._recv = torch.zeros(self.slot * self.world, dtype=torch.int32, device=device)

    def exchange(self, rank: int, owned_words: np.ndarray) -> ExchangeResult:
        import torch

        b, e = self.ranges[rank]
        if owned_words.shape[0] != e - b:
            raise ValueError("owned frontier slice has the wrong length")
        self._send.zero_()
        self._send[: e - b] = torch.from_numpy(owned_words.view(np.int32).copy()).to(self.device)
        self.dist.all_gather_into_tensor(self._recv, self._send, group=self.group)
        gathered = self._recv.cpu().numpy().view(np.uint32)
        frontier = np.zeros(self.n_words, dtype=np.uint32)
        for r, (rb, re) in enumerate(self.ranges):
            frontier[rb:re] = gathered[r * self.slot: r * self.slot + (re - rb)]
        newly = int(np.unpackbits(frontier.view(np.uint8)).sum())
        return ExchangeResult(frontier, newly > 0, newly)


# ---- the device path of chunk-range sharding --------------------------------

class DeviceShard:
    """One rank's shard of a sharded BFS: a device SlimSellRepr (the whole
    layout; this rank sweeps chunks [cb, ce)) driven through the C-ABI
    ssb_bfs_shard_* calls."""

    def __init__(self, r, cb: int, ce: int):
        import torch

        self.r, self.cb, self.ce = r, int(cb), int(ce)
        self.owned = torch.zeros(max(self.ce - self.cb, 1), dtype=torch.int32, device="cuda")

    def begin(self, root: int, opts) -> None:
        import ctypes as C

        from . import _lib as L
        from .api import _check
        o = opts._c()
        _check(L.lib().ssb_bfs_shard_begin(self.r._h, int(root), C.byref(o), self.cb, self.ce))

    def step(self):
        """One iteration over the owned chunks: (local IterStats, owned words)."""
        import ctypes as C

        from . import _lib as L
        from .api import IterStats, _check
        st = L.IterStatsC()
        _check(L.lib().ssb_bfs_shard_step(self.r._h, C.byref(st), C.c_void_p(self.owned.data_ptr())))
        s = IterStats(st.iteration, st.elapsed_ns, st.chunks_processed, st.chunks_skipped,
                      st.subchunks_processed, st.columns_processed, st.frontier_size)
        return s, self.owned[: self.ce - self.cb]

    def launches(self) -> int:
        """Kernels the current/last sharded BFS launched on this rank."""
        import ctypes as C

        from . import _lib as L
        from .api import _check
        ms = C.c_double()
        n = np.zeros(1, np.int64)
        _check(L.lib().ssb_bfs_last_timing(self.r._h, C.byref(ms), n.ctypes.data_as(L.i64p)))
        return int(n[0])

    def exchange(self, full_words, newly_total: int) -> None:
        import ctypes as C

        import torch

        from . import _lib as L
        from .api import _check
        torch.cuda.current_stream().synchronize()
        _check(L.lib().ssb_bfs_shard_exchange(self.r._h, C.c_void_p(full_words.data_ptr()),
                                              int(newly_total)))

    def fetch(self, want_parents: bool, dist: np.ndarray, parent: np.ndarray) -> None:
        from . import _lib as L
        from .api import _check, _p
        _check(L.lib().ssb_bfs_shard_fetch(self.r._h, int(want_parents), _p(dist), _p(parent)))

    # -- asynchronous stepping: no host round trip inside the BFS ------------
    def stream(self):
        """The library stream of this shard's handle as a torch stream: the
        all-gather is enqueued on it between the step and the exchange."""
        import ctypes as C

        import torch

        from . import _lib as L
        from .api import _check
        if getattr(self, "_stream", None) is None:
            p = C.c_void_p()
            _check(L.lib().ssb_graph_stream(self.r._h, C.byref(p)))
            self._stream = torch.cuda.ExternalStream(p.value)
        return self._stream

    def begin_async(self, root: int, opts) -> None:
        import ctypes as C

        from . import _lib as L
        from .api import _check
        o = opts._c()
        _check(L.lib().ssb_bfs_shard_begin_async(self.r._h, int(root), C.byref(o), self.cb, self.ce))

    def step_async(self):
        """Queue one iteration's sweep; returns the owned-words view (filled on
        the shard's stream)."""
        import ctypes as C

        from . import _lib as L
        from .api import _check
        _check(L.lib().ssb_bfs_shard_step_async(self.r._h, C.c_void_p(self.owned.data_ptr())))
        return self.owned[: self.ce - self.cb]

    def exchange_async(self, full_words) -> None:
        import ctypes as C

        from . import _lib as L
        from .api import _check
        _check(L.lib().ssb_bfs_shard_exchange_async(self.r._h, C.c_void_p(full_words.data_ptr())))

    def front(self, k: int) -> int:
        """Global |F_k| (waits for iteration k's exchange only)."""
        from . import _lib as L
        from .api import _check, _p
        out = np.zeros(1, np.int64)
        _check(L.lib().ssb_bfs_shard_front(self.r._h, int(k), _p(out)))
        return int(out[0])

    def finish(self, iterations: int):
        """(this rank's per-iteration counters, device ms of the BFS)."""
        import ctypes as C

        from . import _lib as L
        from .api import _check, _stats_list
        st = (L.IterStatsC * max(iterations, 1))()
        ms = C.c_double()
        _check(L.lib().ssb_bfs_shard_finish(self.r._h, int(iterations), st, int(iterations), C.byref(ms)))
        return _stats_list(st, iterations), float(ms.value)


class P2PUnavailable(RuntimeError):
    """The fused peer exchange cannot be set up on this group of GPUs."""


class P2PShard:
    """One rank's shard of the FUSED multi-GPU BFS: the frontier exchange runs
    inside the BFS kernel over peer-mapped windows (ssb_p2p_* / ssb_bfs_p2p),
    so a BFS is one cooperative launch per rank with no host step between
    iterations. attach() is collective over torch.distributed: the ranks swap
    their windows' CUDA IPC handles (all_gather_object) and map each other's."""

    def __init__(self, r, *segments):
        """segments: (cb, ce), or one list of (cb, ce) segments."""
        self.r = r
        self.segs = _segments_of(segments if len(segments) == 2 else segments[0])

    def window_handle(self) -> bytes:
        import ctypes as C

        from . import _lib as L
        from .api import _check
        h = (C.c_char * 64)()
        nbytes = np.zeros(1, np.int64)
        _check(L.lib().ssb_p2p_window(self.r._h, h, nbytes.ctypes.data_as(L.i64p)))
        return bytes(h)

    def attach(self, rank: int, world: int, handles) -> None:
        import ctypes as C

        from . import _lib as L
        from .api import _check
        if len(handles) != world or any(len(h) != 64 for h in handles):
            raise ValueError("need one 64-byte IPC handle per rank")
        buf = C.create_string_buffer(b"".join(handles), 64 * world)
        b = np.array([x for seg in self.segs for x in seg], dtype=np.int64)
        _check(L.lib().ssb_p2p_attach_segments(self.r._h, int(rank), int(world), buf,
                                               b.ctypes.data_as(L.i64p), len(self.segs)))

    def attach_dist(self, group=None) -> None:
        """Collective: every rank maps every peer's window. A rank that cannot
        (e.g. CUDA IPC refused) makes EVERY rank raise P2PUnavailable, so the
        caller can fall back to the NCCL exchange instead of a hung barrier."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        mine = self.window_handle()
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        err = ""
        try:
            self.attach(rank, world, handles)
        except Exception as e:  # noqa: BLE001 - reported to every rank below
            err = f"rank {rank}: {e}"
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        failed = [x for x in errs if x]
        if failed:
            raise P2PUnavailable("; ".join(failed))
        dist.barrier(group=group)  # every window mapped and zeroed before any BFS

    def run(self, root: int, opts):
        """One BFS (every rank calls it with the same root/opts). Returns
        (iterations, device ms, this rank's per-iteration counters)."""
        import ctypes as C

        from . import _lib as L
        from .api import _check, _stats_list
        o = opts._c()
        cap = 4096
        st = (L.IterStatsC * cap)()
        k = np.zeros(1, np.int64)
        ms = C.c_double()
        rc = L.lib().ssb_bfs_p2p(self.r._h, int(root), C.byref(o), st, cap, k.ctypes.data_as(L.i64p),
                                 C.byref(ms))
        _check(rc)
        if int(k[0]) > cap:  # every rank reruns the same root: the group stays in step
            cap = int(k[0])
            st = (L.IterStatsC * cap)()
            _check(L.lib().ssb_bfs_p2p(self.r._h, int(root), C.byref(o), st, cap,
                                       k.ctypes.data_as(L.i64p), C.byref(ms)))
        return int(k[0]), float(ms.value), _stats_list(st, int(k[0]))

    def fetch(self, want_parents: bool, dist: np.ndarray, parent: np.ndarray) -> None:
        from . import _lib as L
        from .api import _check, _p
        _check(L.lib().ssb_bfs_shard_fetch(self.r._h, int(want_parents), _p(dist), _p(parent)))


def run_p2p_group(reprs, ranges, root: int, opts, fetch: bool = True):
    """The fused multi-GPU BFS with every rank emulated on THIS device: one
    cooperative launch runs all ranks' sweeps and their in-kernel frontier
    exchange (ssb_bfs_p2p_group). Returns (dist, parent, per_iter, device_ms)
    assembled over the shards (dist / parent None when fetch is False)."""
    import ctypes as C

    from . import _lib as L
    from .api import KINF, _check, _p, _stats_list
    world = len(reprs)
    hs = (C.c_void_p * world)(*[r._h for r in reprs])
    segs = [_segments_of(x) for x in ranges]  # per rank: (b, e) or [(b, e), ...]
    rg = np.array([x for sg in segs for seg in sg for x in seg], dtype=np.int64)
    cnt = np.array([len(sg) for sg in segs], dtype=np.int64)
    o = opts._c()
    cap = 4096
    st = (L.IterStatsC * cap)()
    k = np.zeros(1, np.int64)
    ms = C.c_double()
    rc = L.lib().ssb_bfs_p2p_group(hs, world, rg.ctypes.data_as(L.i64p), cnt.ctypes.data_as(L.i64p),
                                   int(root), C.byref(o), st, cap, k.ctypes.data_as(L.i64p), C.byref(ms))
    _check(rc)
    if int(k[0]) > cap:  # deeper than the first buffer: rerun once with room for every record
        cap = int(k[0])
        st = (L.IterStatsC * cap)()
        _check(L.lib().ssb_bfs_p2p_group(hs, world, rg.ctypes.data_as(L.i64p), cnt.ctypes.data_as(L.i64p),
                                         int(root), C.byref(o), st, cap, k.ctypes.data_as(L.i64p),
                                         C.byref(ms)))
    if not fetch:  # the BFS only (results stay on the devices)
        return None, None, _stats_list(st, int(k[0])), float(ms.value)
    n = reprs[0].n
    dist = np.full(n, KINF, dtype=np.int64)
    parent = np.full(n, -1, dtype=np.int64)
    want = bool(opts.want_parents) and int(opts.variant) == 3
    for r in reprs:
        _check(L.lib().ssb_bfs_shard_fetch(r._h, int(want), _p(dist), _p(parent)))
    return dist, (parent if want else parent[:0]), _stats_list(st, int(k[0])), float(ms.value)


class LocalComm:
    """Every shard lives in this process (one GPU emulating several ranks):
    the all-gather is a concatenation in rank order, reductions are sums."""

    def allgather_frontier(self, owned_list):
        import torch
        return torch.cat(list(owned_list)).contiguous()

    def allreduce_sum(self, arrays):
        return np.sum(np.stack(arrays), axis=0)


class TorchComm:
    """One shard per process over torch.distributed (NCCL on B200s): a padded
    all_gather_into_tensor of the owned frontier words, all_reduce for the
    counters."""

    def __init__(self, ranges, group=None):
        import torch.distributed as dist
        self.ranges = ranges
        self.group = group
        self.slot = max(1, max(e - b for b, e in ranges))
        # gloo (functional runs with ranks sharing a GPU) exchanges host tensors
        self.host = dist.get_backend(group) == "gloo"
        # NCCL: the all-gather runs on the caller's current (the shard's) stream,
        # so the BFS steps without host synchronisation (run_sharded_bfs_async)
        self.device_async = not self.host

    def allgather_frontier(self, owned_list):
        import torch
        import torch.distributed as dist
        (owned,) = owned_list
        dev = "cpu" if self.host else owned.device
        send = torch.zeros(self.slot, dtype=torch.int32, device=dev)
        send[: owned.shape[0]] = owned.to(dev)
        recv = torch.empty(self.slot * len(self.ranges), dtype=torch.int32, device=dev)
        if self.host:
            parts = list(recv.split(self.slot))
            dist.all_gather(parts, send, group=self.group)
        else:
            dist.all_gather_into_tensor(recv, send, group=self.group)
        out = torch.cat([recv[r * self.slot: r * self.slot + (e - b)]
                         for r, (b, e) in enumerate(self.ranges)]).contiguous()
        return out.to(owned.device)

    def allreduce_sum(self, arrays):
        import torch
        import torch.distributed as dist
        (a,) = arrays
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64))
        if not self.host:
            t = t.cuda()
        dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()


def _cap_of(opts, n: int, max_iterations: int) -> int:
    """bfs.cpp:70-71: opts.max_iterations > 0 ? it : n + 1 (an explicit
    max_iterations argument overrides)."""
    if max_iterations > 0:
        return max_iterations
    return int(opts.max_iterations) if int(opts.max_iterations) > 0 else n + 1


def _gather_results(shards, opts, n, per_iter, fetch, converged):
    from .api import KINF, BfsCapError, BfsResult
    if not converged:  # bfs.cpp:86-90: the partial distances, no parents
        dist = np.full(n, KINF, dtype=np.int64)
        for sh in shards:
            sh.fetch(False, dist, dist.copy())
        raise BfsCapError(f"BFS did not converge within {len(per_iter)} iterations",
                          BfsResult(dist, dist[:0], len(per_iter), per_iter))
    if not fetch:  # the BFS only (results stay on the devices)
        return None, None, per_iter
    dist = np.full(n, KINF, dtype=np.int64)
    parent = np.full(n, -1, dtype=np.int64)
    want = bool(opts.want_parents) and int(opts.variant) == 3
    for sh in shards:
        sh.fetch(want, dist, parent)
    return dist, (parent if want else parent[:0]), per_iter


def run_sharded_bfs(shards, comm, root: int, opts, max_iterations: int = 0, fetch: bool = True):
    """A BFS over chunk-range shards: per iteration every shard sweeps its
    chunks, the owned frontier words are all-gathered, |newly| is summed, and
    the full frontier is installed on every shard. Returns (dist, parent,
    per_iter) — dist/parent of the rows this process owns (other rows hold the
    sentinels KINF / -1) and the global per-iteration counters. The cap is
    opts.max_iterations (bfs.cpp:70-71); hitting it raises BfsCapError with
    the partial distances and no parents, as bfs_spmv does.

    One shard per process over a device communicator (NCCL): the asynchronous
    form — no host synchronisation inside the BFS (run_sharded_bfs_async).
    Several shards in one process (LocalComm) or a host communicator (gloo)
    step synchronously."""
    if len(shards) == 1 and getattr(comm, "device_async", False):
        return run_sharded_bfs_async(shards[0], comm, root, opts, max_iterations, fetch)
    from .api import IterStats
    for sh in shards:
        sh.begin(root, opts)
    n = shards[0].r.n
    cap = _cap_of(opts, n, max_iterations)
    per_iter = []
    converged = False
    for k in range(1, cap + 1):
        locals_, owned = zip(*[sh.step() for sh in shards])
        counts = comm.allreduce_sum([np.array([s.chunks_processed, s.chunks_skipped,
                                               s.subchunks_processed, s.columns_processed,
                                               s.frontier_size, s.elapsed_ns], dtype=np.int64)
                                     for s in locals_])
        full = comm.allgather_frontier(owned)
        for sh in shards:
            sh.exchange(full, int(counts[4]))
        per_iter.append(IterStats(k, int(counts[5]), *[int(x) for x in counts[:5]]))
        if counts[4] == 0:
            converged = True
            break
    return _gather_results(shards, opts, n, per_iter, fetch, converged)


def run_sharded_bfs_async(shard, comm, root: int, opts, max_iterations: int = 0, fetch: bool = True):
    """The NCCL form without host round trips: sweep (library stream) ->
    all-gather (NCCL, enqueued on the same stream) -> exchange (install +
    device-side |F| count) per iteration; the host only polls |F_{k-1}| while
    iteration k is already queued. The counters stay on the device and are
    all-reduced ONCE at the end of the BFS."""
    import torch

    from .api import IterStats
    n = shard.r.n
    cap = _cap_of(opts, n, max_iterations)
    shard.begin_async(root, opts)
    stream = shard.stream()
    iterations, converged = 0, False
    with torch.cuda.stream(stream):
        for k in range(1, cap + 1):
            owned = shard.step_async()
            full = comm.allgather_frontier([owned])
            shard.exchange_async(full)
            if k >= 2 and shard.front(k - 1) == 0:  # iteration k was queued after convergence: a no-op
                iterations, converged = k - 1, True
                break
        else:
            iterations = cap
            converged = shard.front(cap) == 0
    local, ms = shard.finish(iterations)
    cols = np.array([[s.chunks_processed, s.chunks_skipped, s.subchunks_processed, s.columns_processed,
                      s.frontier_size, s.elapsed_ns] for s in local], dtype=np.int64).reshape(-1, 6)
    tot = comm.allreduce_sum([cols.reshape(-1)]).reshape(-1, 6)  # once per BFS
    per_iter = [IterStats(k + 1, int(r[5]), *[int(x) for x in r[:5]]) for k, r in enumerate(tot)]
    shard.last_ms = ms
    return _gather_results([shard], opts, n, per_iter, fetch, converged)


# ---- one process, several devices (ssb_ctx_*) ------------------------------

class Context:
    """The devices of a single-process multi-GPU job (ssb_ctx_create): all
    distinct — peer access between every pair, one cooperative launch per
    device with the fused NVLink exchange; all the same — the ranks emulated
    as one cooperative launch on that device."""

    def __init__(self, device_ids):
        import ctypes as C

        from . import _lib as L
        from .api import _check
        ids = (C.c_int * len(device_ids))(*[int(d) for d in device_ids])
        h = C.c_void_p()
        _check(L.lib().ssb_ctx_create(len(device_ids), ids, C.byref(h)))
        self._h = h
        self.device_ids = list(device_ids)

    def build(self, g, C_: int = 32, sigma: int | None = None, segments: int = 4) -> "ShardedLayout":
        """The layout of g sharded over the ranks (segments round-robin chunk
        segments per rank)."""
        import ctypes as C

        from . import _lib as L
        from .api import _check
        h = C.c_void_p()
        _check(L.lib().ssb_ctx_build(self._h, g._h, int(C_), int(sigma if sigma is not None else
                                                                 g.num_vertices()), int(segments), C.byref(h)))
        return ShardedLayout(self, h)

    def __del__(self):
        try:
            from . import _lib as L
            L.lib().ssb_ctx_destroy(self._h)
        except Exception:
            pass


class ShardedLayout:
    def __init__(self, ctx: Context, handle):
        import ctypes as C

        from . import _lib as L
        from .api import _check
        self.ctx, self._h = ctx, handle
        world = len(ctx.device_ids)
        nr = C.c_int()
        n = np.zeros(1, np.int64)
        cells = np.zeros(world, np.int64)
        segs = np.zeros(world, np.int64)
        _check(L.lib().ssb_sharded_info(self._h, C.byref(nr), n.ctypes.data_as(L.i64p),
                                        cells.ctypes.data_as(L.i64p), segs.ctypes.data_as(L.i64p)))
        self.n, self.cells_per_rank, self.segments_per_rank = int(n[0]), cells, segs

    def bfs_spmv(self, root: int, opts=None):
        """bfs_spmv (bfs.hpp:80-81) over the shards; BfsResult as bfs_spmv."""
        import ctypes as C

        from . import _lib as L
        from .api import BfsCapError, BfsOptions, BfsResult, _p, _raise, _stats_list
        opts = opts or BfsOptions()
        o = opts._c()
        n = self.n
        dist = np.empty(max(n, 1), np.int64)
        parent = np.empty(max(n, 1), np.int64)
        plen = np.zeros(1, np.int64)
        it = np.zeros(1, np.int64)
        ms = C.c_double()
        cap = min(max(n + 2, 2), 1 << 12)
        while True:
            st = (L.IterStatsC * cap)()
            rc = L.lib().ssb_sharded_bfs(self._h, int(root), C.byref(o), _p(dist), _p(parent), _p(plen), st, cap,
                                         _p(it), C.byref(ms))
            if rc not in (L.SSB_OK, L.SSB_ECAP):
                _raise(rc)
            if int(it[0]) <= cap:
                break
            cap = int(it[0])
        k = int(it[0])
        self.last_ms = float(ms.value)
        res = BfsResult(dist[:n].copy(), parent[: int(plen[0])].copy(), k, _stats_list(st, k))
        if rc == L.SSB_ECAP:
            raise BfsCapError(L.lib().ssb_last_error().decode(), BfsResult(res.dist, res.dist[:0], k, res.per_iter))
        return res

    def __del__(self):
        try:
            from . import _lib as L
            L.lib().ssb_sharded_destroy(self._h)
        except Exception:
            pass
