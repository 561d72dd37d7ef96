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
