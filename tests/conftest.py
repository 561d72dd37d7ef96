import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: larger graphs (still minutes at most)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle import Port, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build(ref=False)
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Reference()


@pytest.fixture(scope="session")
def ssb():
    """The product package with its CUDA library loaded (GPU tests only)."""
    import paper_2010_09913_b200 as ssb
    ssb.lib()
    return ssb


@pytest.fixture(scope="session")
def edge_graphs(port):
    """Edge cases the reference's own tests do not enumerate: one vertex, no
    edges, self loops only (dropped by from_pairs, graph.cpp:16-40), two
    components, and n just around multiples of C = 32 (ragged last chunk) with
    duplicate pairs and loops mixed in. (name, n, normalized uv) triples."""
    import numpy as np
    rng = np.random.default_rng(5)
    none = np.zeros((0, 2), np.int64)
    cliques = [[i, j] for a in (0, 6) for i in range(a, a + 6) for j in range(a, a + 6) if i != j]
    out = [("single", 1, none), ("edgeless5", 5, none),
           ("loops_only4", *port.from_pairs(np.stack([np.arange(4)] * 2, 1), 4)),
           ("two_cliques", *port.from_pairs(np.array(cliques), 12))]
    for n in (31, 32, 33, 65, 97):
        pairs = rng.integers(0, n, size=(3 * n, 2))
        pairs = np.concatenate([pairs, pairs[: n // 3], np.stack([np.arange(0, n, 5)] * 2, 1)])
        out.append((f"ragged{n}", *port.from_pairs(pairs, n)))
    return out
