"""Canonical digests of integer plan/partition structures.

Shared by ``make_golden.py`` (run against the reference) and the tests
(run against the oracle and the package) so that large integer structures
are pinned by a short sha256 instead of a bulky fixture.
"""

import hashlib
import json

import numpy as np


def _arr(h, a):
    a = np.ascontiguousarray(np.asarray(a, dtype="<i8"))
    h.update(len(a).to_bytes(8, "little"))
    h.update(a.tobytes())


def plan_digest(m, n, N, U, T, carry, load, fetch, nbr_carry, live, slots,
                caps, volumes):
    """fetch[i][j] is a mapping peer k -> array; slots[i][j] is aligned
    with live[i][j]."""
    h = hashlib.sha256()
    h.update(json.dumps([int(m), int(n), [int(c) for c in caps],
                         [int(v) for v in volumes]]).encode())
    for j in range(n):
        _arr(h, U[j])
    for i in range(m):
        for j in range(n):
            for a in (N[i][j], T[i][j], carry[i][j], load[i][j],
                      nbr_carry[i][j], live[i][j], slots[i][j]):
                _arr(h, a)
            for k in sorted(fetch[i][j]):
                h.update(int(k).to_bytes(8, "little"))
                _arr(h, fetch[i][j][k])
    return h.hexdigest()


def chunk_digest(chunks):
    """chunks: grid[i][j] of mappings/objects with the ChunkSubgraph fields."""
    h = hashlib.sha256()
    for row in chunks:
        for c in row:
            get = (lambda k: c[k]) if isinstance(c, dict) else (lambda k: getattr(c, k))
            for k in ("vertices", "sources", "csc_offsets", "csc_local_src",
                      "csr_offsets", "csr_local_dst", "csr_edge_perm"):
                _arr(h, get(k))
            w = np.ascontiguousarray(np.asarray(get("edge_weights"), dtype="<f8"))
            h.update(w.tobytes())
    return h.hexdigest()
