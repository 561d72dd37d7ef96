"""Root selection and result fingerprints shared by bench.py, the tests and
the golden-vector generator. Pure numpy / torch: importing this module loads
no shared library (the bench's reference arm uses it too).

* ``graph500_roots`` — the reference's ``pick_roots`` stream (cli.cpp:114-134:
  ``SplitMix64(seed).split(0x526f)``, ``next() % n``, distinct) additionally
  rejecting degree-0 vertices.
* ``ph64`` — an order-sensitive, PARALLEL fingerprint of an int64 vector:
  ``Σ_i mix64(v[i] + (i+1)·γ) mod 2^64`` (γ = 0x9E3779B97F4A7C15, mix64 the
  SplitMix64 finaliser, generator.hpp:12-20). FNV-1a (the golden files' other
  fingerprint) is byte-serial; this one is computed on the device in
  milliseconds, so bench.py can compare every root of an S26 step with the
  reference's output recorded in ``tests/golden/golden_big.json``.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
K1, K2 = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def mix64(x: int) -> int:
    x = ((x ^ (x >> 30)) * K1) & M64
    x = ((x ^ (x >> 27)) * K2) & M64
    return x ^ (x >> 31)


def graph500_roots(deg: np.ndarray, want: int, seed: int) -> list[int]:
    """pick_roots' stream (cli.cpp:114-134) rejecting degree-0 vertices;
    ``deg`` is indexed by ORIGINAL vertex id."""
    n = int(deg.shape[0])
    s = mix64(seed ^ mix64((0x526F + 0x6A09E667F3BCC909) & M64))
    out, seen = [], set()
    limit = min(want, int(np.count_nonzero(deg)))
    while len(out) < limit:
        s = (s + GAMMA) & M64
        r = mix64(s) % n
        if r not in seen:
            seen.add(r)
            if deg[r] > 0:
                out.append(int(r))
    return out


def ph64_np(v: np.ndarray, block: int = 1 << 24) -> str:
    """ph64 of an int64 vector on the host (numpy, uint64 wrap-around)."""
    v = np.ascontiguousarray(v, dtype=np.int64).view(np.uint64)
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for b in range(0, v.shape[0], block):
            x = v[b:b + block] + (np.arange(b + 1, b + 1 + min(block, v.shape[0] - b), dtype=np.uint64)
                                  * np.uint64(GAMMA))
            x = (x ^ (x >> np.uint64(30))) * np.uint64(K1)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(K2)
            x = x ^ (x >> np.uint64(31))
            total = total + x.sum(dtype=np.uint64)
    return format(int(total), "016x")


def _as_signed(c: int) -> int:
    return c - (1 << 64) if c >= 1 << 63 else c


def ph64_torch(t) -> str:
    """ph64 of an int64 torch tensor on its own device. int64 arithmetic wraps
    mod 2^64 like uint64; logical right shifts are arithmetic shifts masked."""
    import torch

    t = t.reshape(-1).to(torch.int64)
    i = torch.arange(1, t.numel() + 1, dtype=torch.int64, device=t.device)
    x = t + i * _as_signed(GAMMA)
    x = (x ^ ((x >> 30) & ((1 << 34) - 1))) * _as_signed(K1)
    x = (x ^ ((x >> 27) & ((1 << 37) - 1))) * _as_signed(K2)
    x = x ^ ((x >> 31) & ((1 << 33) - 1))
    return format(int(x.sum().item()) & M64, "016x")


def ph64_partial_torch(t, mask) -> int:
    """The ph64 terms of the positions where `mask` holds, summed mod 2^64 as a
    signed int64 (ph64 is a sum over positions, so ranks that own disjoint
    rows add their partials — one all-reduce instead of gathering the vector)."""
    import torch

    t = t.reshape(-1).to(torch.int64)
    i = torch.arange(1, t.numel() + 1, dtype=torch.int64, device=t.device)
    x = t + i * _as_signed(GAMMA)
    x = (x ^ ((x >> 30) & ((1 << 34) - 1))) * _as_signed(K1)
    x = (x ^ ((x >> 27) & ((1 << 37) - 1))) * _as_signed(K2)
    x = x ^ ((x >> 31) & ((1 << 33) - 1))
    return _as_signed(int(x[mask.reshape(-1)].sum().item()) & M64)


def ph64_format(total: int) -> str:
    return format(int(total) & M64, "016x")
