"""Initial store contents (the Heap's materialisation rule plus injections).

Default rule, restated from ``Heap.get`` (``executor.py:54-61``): a store
materialises as ``default_rng([seed, sid]).integers(1, 10, size=shape)``
converted to float64.  Re-materialising after ``free`` gives identical
contents (``test_executor.py:40-46``).

Harness traces inject other contents by store id (SURVEY §7.1 "InitHeap"):
zero reduction targets, a constant, a seeded uniform field, or the tiles of a
2-D Poisson matrix in the per-tile CSR layout used by ``SPMV_CSR``.  Both the
CPU reference run and the GPU run call :func:`host_contents` on the same spec,
so their starting heaps are identical.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


def default_contents(seed: int, sid: int, shape: Sequence[int]) -> np.ndarray:
    rng = np.random.default_rng([seed, sid])
    return rng.integers(1, 10, size=tuple(shape)).astype(np.float64)


def poisson_tile_layout(nx: int, ny: int, k: int) -> dict:
    """Row bands of the 5-point Laplacian on an ``nx`` x ``ny`` grid, ``k`` tiles."""
    if ny % k:
        raise ValueError(f"grid rows {ny} must be divisible by tiles {k}")
    n = nx * ny
    t = n // k
    # every tile has the same nnz except the first and last (one grid row each
    # loses its north / south neighbour); pad to the maximum
    per_row_interior = 5 * nx - 2
    nnz_full = (ny // k) * per_row_interior
    # tile 0 holds the top grid row and tile k-1 the bottom one; each loses nx
    nnz_max = nnz_full - (2 * nx if k == 1 else nx if k == 2 else 0)
    return {"nx": nx, "ny": ny, "k": k, "n": n, "t": t, "nnz_max": nnz_max}


def poisson_tile(nx: int, ny: int, k: int, p: int, dtype_idx=np.float64):
    """(rowptr[t+1], cols[nnz_max], vals[nnz_max]) of tile ``p``; columns global."""
    lay = poisson_tile_layout(nx, ny, k)
    t, nnz_max = lay["t"], lay["nnz_max"]
    r = np.arange(p * t, (p + 1) * t, dtype=np.int64)
    iy, ix = r // nx, r % nx
    cand = np.stack([r - nx, r - 1, r, r + 1, r + nx], axis=1)
    ok = np.stack([iy > 0, ix > 0, np.ones_like(ix, dtype=bool), ix < nx - 1, iy < ny - 1], axis=1)
    coef = np.broadcast_to(np.array([-1.0, -1.0, 4.0, -1.0, -1.0]), cand.shape)
    cols = cand[ok]
    vals = coef[ok]
    counts = ok.sum(axis=1)
    rowptr = np.zeros(t + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    c = np.zeros(nnz_max, dtype=np.int64)
    v = np.zeros(nnz_max, dtype=np.float64)
    c[: cols.size] = cols
    v[: vals.size] = vals
    return rowptr.astype(dtype_idx), c.astype(dtype_idx), v


def row_chunks(spec: dict | None, seed: int, sid: int, shape: Sequence[int], row_end: int, chunk_elems: int = 1 << 24):
    """Yield ``(row0, row1, rows)`` of the initial contents, dim-0 rows ``[0, row_end)``.

    The RNG kinds are generated as one sequential stream in bounded chunks
    (numpy's Generator continues its stream across calls, so the chunks
    concatenate to exactly ``host_contents``).  Rank-0 stores yield one chunk.
    """
    shape = tuple(shape)
    if not shape:
        yield 0, 1, host_contents(spec, seed, sid, shape)
        return
    row = 1
    for e in shape[1:]:
        row *= e
    step = max(1, chunk_elems // max(row, 1))
    kind = None if spec is None else spec["kind"]
    if kind is None or kind == "uniform":
        if kind is None:
            rng = np.random.default_rng([seed, sid])
            draw = lambda n: rng.integers(1, 10, size=n).astype(np.float64)  # noqa: E731
        else:
            rng = np.random.default_rng([int(spec.get("seed", 0)), int(spec.get("key", sid))])
            scale = float(spec["scale"]) if "scale" in spec else None

            def draw(n):
                a = rng.random(size=n, dtype=np.float64)
                if scale is not None:
                    a *= scale
                return a

        for r0 in range(0, row_end, step):
            r1 = min(row_end, r0 + step)
            yield r0, r1, draw((r1 - r0) * row).reshape((r1 - r0,) + shape[1:])
        return
    if kind in ("zeros", "const", "poisson_invdiag"):
        v = {"zeros": 0.0, "poisson_invdiag": 0.25}.get(kind, float(spec.get("value", 0.0)))
        for r0 in range(0, row_end, step):
            r1 = min(row_end, r0 + step)
            yield r0, r1, np.full((r1 - r0,) + shape[1:], v, dtype=np.float64)
        return
    full = host_contents(spec, seed, sid, shape)
    yield 0, row_end, full[:row_end]


def host_contents(spec: dict | None, seed: int, sid: int, shape: Sequence[int]) -> np.ndarray:
    """float64 host array for store ``sid`` under an init spec (None = default rule)."""
    shape = tuple(shape)
    if spec is None:
        return default_contents(seed, sid, shape)
    kind = spec["kind"]
    if kind == "zeros":
        return np.zeros(shape, dtype=np.float64)
    if kind == "const":
        return np.full(shape, float(spec["value"]), dtype=np.float64)
    if kind == "uniform":
        rng = np.random.default_rng([int(spec.get("seed", 0)), int(spec.get("key", sid))])
        out = rng.random(size=shape, dtype=np.float64)
        if "scale" in spec:
            out *= float(spec["scale"])
        return out
    if kind in ("csr_rowptr", "csr_cols", "csr_vals"):
        nx, ny, k = int(spec["nx"]), int(spec["ny"]), int(spec["k"])
        which = ("csr_rowptr", "csr_cols", "csr_vals").index(kind)
        out = np.zeros(shape, dtype=np.float64).reshape(k, -1)
        for p in range(k):
            out[p, :] = poisson_tile(nx, ny, k, p)[which]
        return out.reshape(shape)
    if kind == "poisson_invdiag":
        return np.full(shape, 0.25, dtype=np.float64)
    raise ValueError(f"unknown init kind {kind!r}")
