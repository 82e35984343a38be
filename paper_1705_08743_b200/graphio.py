"""Edge-list graphs -> device matrices (drop-in for semimat.graphio).

Text format (pkg/src/semimat/graphio.py:1-6): a header line ``p <count>``,
then one edge per line, ``u v`` or ``u v w`` (weight 1 when omitted); ``#``
starts a comment and blank lines are skipped.  ``parse_edge_list`` checks the
same things in the same order and raises the same ``GraphParseError``
messages with the offending line number (graphio.py:32-79); the builders
hand the edge list to the device constructors (graphio.py:82-95):
``from_edges`` scatters it on the GPU (csrc/construct.cu), and the Boolean
adjacency is packed from one host array instead of one ``set`` per edge.
Parsing is host work: text is not on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .antidist import AntidistMatrix, DistMatrix
from .boolmat import BoolMatrix

__all__ = ["GraphParseError", "GraphSpec", "parse_edge_list", "bool_adjacency", "antidist_adjacency",
           "dist_adjacency"]


class GraphParseError(ValueError):
    """Malformed edge-list text; ``lineno`` is the 1-based offending line, or None."""

    def __init__(self, message, lineno=None):
        super().__init__(message if lineno is None else f"line {lineno}: {message}")
        self.lineno = lineno


@dataclass
class GraphSpec:
    """A parsed directed graph: vertex count, (u, v, w) edges in file order,
    and whether any edge carried an explicit weight."""

    vertex_count: int
    edges: list[tuple[int, int, int]] = field(default_factory=list)
    weighted: bool = False


def _records(text: str):
    """(line number, fields) of every line that is not blank or all comment."""
    for lineno, raw in enumerate(text.splitlines(), 1):
        body = raw.partition("#")[0]
        fields = body.split()
        if fields:
            yield lineno, body.strip(), fields


def _header(lineno: int, fields: list[str]) -> int:
    if len(fields) != 2 or fields[0] != "p":
        raise GraphParseError("expected header 'p <vertex_count>'", lineno)
    try:
        count = int(fields[1])
    except ValueError:
        raise GraphParseError(f"vertex count {fields[1]!r} is not an integer", lineno) from None
    if count < 1:
        raise GraphParseError(f"vertex count must be positive, got {count}", lineno)
    return count


def _edge(lineno: int, line: str, fields: list[str], count: int) -> tuple[int, int, int, bool]:
    if not 2 <= len(fields) <= 3:
        raise GraphParseError(f"expected 'u v [w]', got {line!r}", lineno)
    try:
        nums = list(map(int, fields))
    except ValueError:
        raise GraphParseError(f"non-integer field in {line!r}", lineno) from None
    for name, x in (("source", nums[0]), ("target", nums[1])):
        if x < 0 or x >= count:
            raise GraphParseError(f"{name} vertex {x} out of range [0, {count})", lineno)
    if len(nums) == 2:
        return nums[0], nums[1], 1, False
    if nums[2] < 0:
        raise GraphParseError(f"negative weight {nums[2]}", lineno)
    return nums[0], nums[1], nums[2], True


def parse_edge_list(text: str) -> GraphSpec:
    """Parse edge-list text into a validated GraphSpec.  Whether a weight fits
    a lane width is checked when a matrix is built (``from_edges``)."""
    records = _records(text)
    first = next(records, None)
    if first is None:
        raise GraphParseError("missing 'p <vertex_count>' header")
    spec = GraphSpec(_header(first[0], first[2]))
    for lineno, line, fields in records:
        u, v, w, explicit = _edge(lineno, line, fields, spec.vertex_count)
        spec.edges.append((u, v, w))
        spec.weighted |= explicit
    return spec


def bool_adjacency(spec: GraphSpec) -> BoolMatrix:
    """Unweighted adjacency: bit (u, v) set for every edge."""
    n = spec.vertex_count
    adj = np.zeros((n, n), dtype=bool)
    if spec.edges:
        e = np.asarray(spec.edges, dtype=np.int64)
        adj[e[:, 0], e[:, 1]] = True
    return BoolMatrix.from_numpy(adj)


def antidist_adjacency(spec: GraphSpec, width: int = 8) -> AntidistMatrix:
    """Weighted adjacency in the anti-distance encoding (built on the device)."""
    return AntidistMatrix.from_edges(spec.vertex_count, spec.edges, width)


def dist_adjacency(spec: GraphSpec, width: int = 8) -> DistMatrix:
    """Weighted adjacency in the plain-distance encoding (built on the device)."""
    return DistMatrix.from_edges(spec.vertex_count, spec.edges, width)
