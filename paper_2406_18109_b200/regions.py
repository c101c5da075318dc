"""Half-open N-d rectangles and disjoint rect lists (host-side coherence algebra).

A Rect is ``(lo, hi)`` with ``lo``/``hi`` integer tuples, as in the reference
``Rect`` (ir.py:193-238).  Lists are kept pairwise disjoint so volumes add.
"""

from __future__ import annotations

from typing import Iterable, Sequence

Rect = tuple[tuple[int, ...], tuple[int, ...]]


def empty(r: Rect) -> bool:
    return any(h <= l for l, h in zip(*r))


def volume(r: Rect) -> int:
    v = 1
    for l, h in zip(*r):
        v *= max(0, h - l)
    return v


def intersect(a: Rect, b: Rect) -> Rect:
    return (
        tuple(max(x, y) for x, y in zip(a[0], b[0])),
        tuple(min(x, y) for x, y in zip(a[1], b[1])),
    )


def overlaps(a: Rect, b: Rect) -> bool:
    return not empty(a) and not empty(b) and not empty(intersect(a, b))


def contains(outer: Rect, inner: Rect) -> bool:
    if empty(inner):
        return True
    return all(ol <= il and ih <= oh for ol, oh, il, ih in zip(outer[0], outer[1], inner[0], inner[1]))


def subtract(a: Rect, b: Rect) -> list[Rect]:
    """a minus b as at most 2*rank disjoint rects."""
    if empty(a):
        return []
    c = intersect(a, b)
    if empty(c):
        return [a]
    out: list[Rect] = []
    lo, hi = list(a[0]), list(a[1])
    for d in range(len(lo)):
        if lo[d] < c[0][d]:
            nlo, nhi = list(lo), list(hi)
            nhi[d] = c[0][d]
            out.append((tuple(nlo), tuple(nhi)))
        if c[1][d] < hi[d]:
            nlo, nhi = list(lo), list(hi)
            nlo[d] = c[1][d]
            out.append((tuple(nlo), tuple(nhi)))
        lo[d], hi[d] = c[0][d], c[1][d]
    return out


def subtract_all(rects: Iterable[Rect], b: Rect) -> list[Rect]:
    out: list[Rect] = []
    for r in rects:
        out.extend(subtract(r, b))
    return out


def minus(rects: Sequence[Rect], cut: Sequence[Rect]) -> list[Rect]:
    out = [r for r in rects if not empty(r)]
    for c in cut:
        if not out:
            break
        out = subtract_all(out, c)
    return out


def _try_merge(a: Rect, b: Rect) -> Rect | None:
    diff = [d for d in range(len(a[0])) if (a[0][d], a[1][d]) != (b[0][d], b[1][d])]
    if len(diff) != 1:
        return None if diff else a
    d = diff[0]
    if a[1][d] == b[0][d]:
        return (a[0], tuple(b[1][i] if i == d else a[1][i] for i in range(len(a[0]))))
    if b[1][d] == a[0][d]:
        return (b[0], tuple(a[1][i] if i == d else b[1][i] for i in range(len(a[0]))))
    return None


def coalesce(rects: list[Rect]) -> list[Rect]:
    rects = [r for r in rects if not empty(r)]
    changed = True
    while changed and len(rects) > 1:
        changed = False
        for i in range(len(rects)):
            for j in range(i + 1, len(rects)):
                m = _try_merge(rects[i], rects[j])
                if m is not None:
                    rects[i] = m
                    rects.pop(j)
                    changed = True
                    break
            if changed:
                break
    return rects


def add(rects: list[Rect], r: Rect) -> list[Rect]:
    if empty(r):
        return rects
    return coalesce(subtract_all(rects, r) + [r])


def covered(rects: Sequence[Rect], r: Rect) -> bool:
    return not minus([r], rects)


def bbox_flat(shape: Sequence[int], r: Rect) -> tuple[int, int]:
    """[first, last+1) row-major element span touched by a non-empty rect."""
    if not shape:
        return (0, 1)
    strides = [1] * len(shape)
    for d in range(len(shape) - 2, -1, -1):
        strides[d] = strides[d + 1] * shape[d + 1]
    first = sum(l * s for l, s in zip(r[0], strides))
    last = sum((h - 1) * s for h, s in zip(r[1], strides))
    return first, last + 1
