"""Edge-list parsing (graphio): the reference's format, validation order and
messages (pkg/src/semimat/graphio.py:32-79; its tests in
pkg/tests/test_graphio.py), checked on CPU; the device builders
(graphio.py:82-95) on the GPU against host-built adjacencies."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1705_08743_b200 import GraphParseError, parse_edge_list
from paper_1705_08743_b200 import graphio


def test_parse_weighted_unweighted_comments():
    spec = parse_edge_list("p 3\n0 1 3\n1 2 4\n")
    assert (spec.vertex_count, spec.edges, spec.weighted) == (3, [(0, 1, 3), (1, 2, 4)], True)
    spec = parse_edge_list("p 2\n0 1\n")
    assert (spec.edges, spec.weighted) == ([(0, 1, 1)], False)
    spec = parse_edge_list("# a graph\n\n  p 4   # four vertices\n0 3 # edge\n\n3 0 0\n  # end\n")
    assert (spec.vertex_count, spec.edges, spec.weighted) == (4, [(0, 3, 1), (3, 0, 0)], True)
    assert parse_edge_list("p 1\n").edges == []


@pytest.mark.parametrize("text,pattern,lineno", [
    ("p 2\n0 5 1\n", r"^line 2: target vertex 5 out of range \[0, 2\)$", 2),
    ("p 2\n7 5 1\n", r"^line 2: source vertex 7 out of range \[0, 2\)$", 2),
    ("p 2\n-1 0\n", r"source vertex -1 out of range", 2),
    ("0 1\n", r"^line 1: expected header 'p <vertex_count>'$", 1),
    ("p 2 3\n", r"expected header", 1),
    ("", r"^missing 'p <vertex_count>' header$", None),
    ("# only a comment\n\n", r"missing 'p <vertex_count>' header", None),
    ("p 2\n0 x\n", r"^line 2: non-integer field in '0 x'$", 2),
    ("p 2\n0 1 -3\n", r"^line 2: negative weight -3$", 2),
    ("p 2\n0 1 2 3\n", r"^line 2: expected 'u v \[w\]', got '0 1 2 3'$", 2),
    ("p 2\n0\n", r"expected 'u v \[w\]', got '0'", 2),
    ("p 0\n", r"^line 1: vertex count must be positive, got 0$", 1),
    ("p x\n", r"^line 1: vertex count 'x' is not an integer$", 1),
    ("\n\np 2\n0 1\n1 9 # far\n", r"^line 5: target vertex 9", 5),
])
def test_parse_errors_match_reference(text, pattern, lineno):
    with pytest.raises(GraphParseError, match=pattern) as ei:
        parse_edge_list(text)
    assert ei.value.lineno == lineno
    assert isinstance(ei.value, ValueError)


@pytest.mark.gpu
def test_builders_on_device(oracle_lib):
    rng = np.random.default_rng(5)
    n = 300
    edges = [(int(u), int(v), int(w)) for u, v, w in zip(rng.integers(0, n, 2000), rng.integers(0, n, 2000),
                                                          rng.integers(0, 200, 2000))]
    text = f"p {n}\n" + "\n".join(f"{u} {v} {w}" for u, v, w in edges) + "\n"
    spec = parse_edge_list(text)
    b = graphio.bool_adjacency(spec)
    want = np.zeros((n, n), dtype=bool)
    for u, v, _ in edges:
        want[u, v] = True
    assert b.to_lists() == want.astype(int).tolist()
    for width in (8, 16, 32):
        lim = (1 << width) - 1
        best = np.full((n, n), lim + 1, dtype=np.int64)
        for u, v, w in edges:
            best[u, v] = min(best[u, v], w)
        d = graphio.dist_adjacency(spec, width)
        a = graphio.antidist_adjacency(spec, width)
        dist = np.where(best > lim, lim, best)
        assert d.to_lists() == dist.tolist()
        assert a.to_lists() == np.where(best > lim, 0, lim - dist).tolist()
    with pytest.raises(ValueError, match=r"weight 300 outside \[0, 255\]"):
        graphio.antidist_adjacency(parse_edge_list("p 2\n0 1 300\n"), 8)
