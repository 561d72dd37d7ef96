"""Edge-list / MatrixMarket ingest (graph.cpp:94-210) against the reference's
own parsers (oracle/_ref): the same graphs, and the same error kind and
message for malformed input. Host-only parsing: runs without a GPU."""
import numpy as np
import pytest

import paper_2010_09913_b200 as ssb
from oracle.cpu import OracleError

CODE = {ssb.InvalidArgument: 1, ssb.OutOfRange: 2, ssb.ParseError: 6}

EDGE_LISTS = [
    b"", b"\n", b"# only a comment\n", b"0 1\n1 2\n2 0\n", b"0 1\r\n1 2\r\n", b"  3   4  \n\t5 6\n",
    b"H 10 2\n0 1\n1 2\n", b"% c\nH 3 1\n# c\n0 1", b"0 0\n1 1\n", b"5 3\n3 5\n5 3\n",
    b"0 1\nH 3 1\n", b"H 3 1\nH 3 1\n", b"H 3\n", b"0 1 2\n", b"0\n", b"0 x\n", b"-1 2\n", b"+1 2\n",
    b"0 1\n99999999999999999999 1\n", b"9223372036854775808 1\n", b"9223372036854775807 0\n" * 0,
    b"H 2 1\n0 5\n", b"0 1\n\n\n2 3\n   \n", b"1 2 # trailing comment\n", b"#0 1\n%2 3\n",
]
ASYM = [b"0 1\n1 0\n", b"0 1\n", b"0 1\n1 0\n2 3\n", b"2 2\n", b"0 1\n1 0\n1 2\n2 1\n0 1\n"]
MM = [
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n2 3\n",
    b"%%MatrixMarket matrix coordinate pattern symmetric\n% comment\n4 4 3\n1 2\n2 3\n4 4\n",
    b"%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 0.5\n3 1 -2\n",
    b"%%MatrixMarket matrix coordinate real symmetric\r\n2 2 1\r\n2 1 1.0\r\n",
    b"", b"hello\n", b"%%MatrixMarket matrix array real general\n", b"%%MatrixMarket matrix coordinate complex general\n",
    b"%%MatrixMarket matrix coordinate pattern hermitian\n", b"%%MatrixMarket matrix coordinate pattern general\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 4 1\n1 2\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2 3\n",
    b"%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 2\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 4\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2\n2 3\n",
    b"%%MatrixMarket matrix coordinate pattern general\n3 3 0\n",
    b"%%MatrixMarket matrix\n", b"%%MatrixMarket matrix coordinate pattern general\n3 3 1\nx 2\n",
]


def ours(fn, text, *args):
    try:
        n, uv = fn(text, *args)
        return ("ok", n, uv)
    except (ssb.InvalidArgument, ssb.OutOfRange, ssb.ParseError) as e:
        return ("err", CODE[type(e)], str(e))


def theirs(fn, text, *args):
    try:
        g = fn(text, *args)
        return ("ok", g.n, g.edges())
    except OracleError as e:
        return ("err", e.code, str(e).split(": ", 1)[1])


def same(port, a, b, text):
    assert a[0] == b[0], (text, a, b)
    if a[0] == "err":
        assert a[1] == b[1] and a[2] == b[2], (text, a, b)
        return
    try:  # normalisation (Graph::from_pairs) — the reference may reject here
        n, uv = port.from_pairs(a[2], a[1])
    except OracleError as e:
        raise AssertionError((text, "from_pairs rejected", e))
    assert n == b[1] and np.array_equal(uv, b[2]), text


@pytest.mark.parametrize("text", EDGE_LISTS)
def test_edge_list_matches_reference(ref, port, text):
    a, b = ours(ssb.parse_edge_list, text), theirs(ref.from_edge_list, text)
    if a[0] == "ok" and b[0] == "err":  # errors raised by from_pairs (e.g. id beyond H n)
        with pytest.raises(OracleError) as e:
            port.from_pairs(a[2], a[1])
        assert e.value.code == b[1]
        return
    same(port, a, b, text)


@pytest.mark.parametrize("text", ASYM)
def test_edge_list_reject_asymmetric_matches_reference(ref, port, text):
    same(port, ours(ssb.parse_edge_list, text, True), theirs(ref.from_edge_list, text, True), text)


@pytest.mark.parametrize("text", MM)
def test_matrix_market_matches_reference(ref, port, text):
    same(port, ours(ssb.parse_matrix_market, text), theirs(ref.from_matrix_market, text), text)


def test_random_texts_match_reference(ref, port):
    rng = np.random.default_rng(7)
    for trial in range(20):
        n = int(rng.integers(1, 200))
        m = int(rng.integers(0, 400))
        uv = rng.integers(0, n, size=(m, 2))
        lines = []
        if trial % 3 == 0:
            lines.append(f"H {n} {m}")
        for u, v in uv:
            if rng.random() < 0.1:
                lines.append("# noise" if rng.random() < 0.5 else "")
            sep = " " * int(rng.integers(1, 4)) if rng.random() < 0.7 else "\t"
            lines.append(f"{u}{sep}{v}")
        eol = "\r\n" if trial % 4 == 1 else "\n"
        text = eol.join(lines).encode()
        same(port, ours(ssb.parse_edge_list, text), theirs(ref.from_edge_list, text), trial)
        sym = trial % 2 == 0
        body = [f"%%MatrixMarket matrix coordinate {'pattern' if trial % 3 else 'real'} "
                f"{'symmetric' if sym else 'general'}", f"{n} {n} {m}"]
        body += [f"{u + 1} {v + 1}" + ("" if trial % 3 else " 1.5") for u, v in uv]
        text = "\n".join(body).encode()
        same(port, ours(ssb.parse_matrix_market, text), theirs(ref.from_matrix_market, text), trial)
