"""Seeded synthetic MaxCut graphs for benchmarks and scaling runs.

* ``random_sparse`` -- uniform random simple graph with about n*deg/2 unit
  edges (BASELINE configs: "synthetic random sparse graph, avg degree ~6").
* ``path_like`` -- a long random path plus sparse chords (degree ~2.2), the shape of
  the paper's largest instance (kmer_A2a, 1.7e8 nodes).
* ``delaunay_like`` -- triangulated periodic lattice with randomly permuted
  vertex labels: every vertex has degree 6 like a planar Delaunay mesh
  (the paper's 10^7-scale instances are delaunay_n23/n24), no locality.

Edges are returned sorted by (u, v) with u < v, which lets ``build_maxcut``
take its linear-time ordering path.
"""

from __future__ import annotations

import numpy as np

from .problem import GraphEdgeList, unique_sorted


def _finish(n, u, v, rng, target=None):
    a = np.minimum(u, v)
    b = np.maximum(u, v)
    keep = a != b
    code = unique_sorted(a[keep] * n + b[keep])
    if target is not None and code.size > target:
        code = np.sort(rng.choice(code, size=target, replace=False))
    return GraphEdgeList(n, code // n, code % n, np.ones(code.size))


def random_sparse(n, deg=6.0, seed=0):
    rng = np.random.default_rng(seed)
    me = int(round(n * deg / 2))
    # loops and repeats are dropped (a ~deg/n fraction), so |E| is just under n*deg/2
    u = rng.integers(0, n, size=me, dtype=np.int64)
    v = rng.integers(0, n, size=me, dtype=np.int64)
    return _finish(n, u, v, rng)


def delaunay_like(n, seed=0):
    rng = np.random.default_rng(seed)
    side = int(round(np.sqrt(n)))
    n = side * side
    i, j = np.divmod(np.arange(n, dtype=np.int64), side)
    vid = lambda a, b: (a % side) * side + (b % side)  # noqa: E731
    u = np.concatenate([np.arange(n, dtype=np.int64)] * 3)
    v = np.concatenate([vid(i, j + 1), vid(i + 1, j), vid(i + 1, j + 1)])
    perm = rng.permutation(n).astype(np.int64)
    return _finish(n, perm[u], perm[v], rng)


def path_like(n, extra=0.1, seed=0):
    """A k-mer-graph-like instance (the paper's 1.7e8-node kmer_A2a family is mostly long
    chains): one path through all n vertices in a random order, plus ``extra * n`` random
    chords; average degree ~ 2 + 2 extra, no locality in the labels."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n).astype(np.int64)
    me = int(round(extra * n))
    u = np.concatenate([perm[:-1], rng.integers(0, n, size=me, dtype=np.int64)])
    v = np.concatenate([perm[1:], rng.integers(0, n, size=me, dtype=np.int64)])
    return _finish(n, u, v, rng)


GENERATORS = {"random_sparse": random_sparse, "delaunay_like": delaunay_like, "path_like": path_like}


def random_completion(n2, n1, m, rank=2, seed=0):
    """Seeded matrix-completion instance (BASELINE configs[3] family): m distinct
    observed entries (i, j) of an n2 x n1 rank-`rank` matrix M = A B^T."""
    from .problem import ObservationSet
    rng = np.random.default_rng(seed)
    draw = int(m * 1.1) + 16
    code = unique_sorted(rng.integers(0, n2, size=draw, dtype=np.int64) * n1
                         + rng.integers(0, n1, size=draw, dtype=np.int64))
    if code.size > m:
        code = np.sort(rng.choice(code, size=m, replace=False))
    i, j = code // n1, code % n1
    A = rng.standard_normal((n2, rank))
    B = rng.standard_normal((n1, rank))
    vals = np.einsum("kr,kr->k", A[i], B[j])
    return ObservationSet(n2, n1, i, j, vals)


GENERATORS["random_completion"] = random_completion
