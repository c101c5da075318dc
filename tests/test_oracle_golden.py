"""Pin the CPU oracle against the reference's own outputs (golden fixtures)."""

import numpy as np
import pytest

from conftest import golden_arrays, same_bits
from oracle.interp import OracleHeap, replay, spmv_csr_rows
from paper_2406_18109_b200.initheap import poisson_tile
from paper_2406_18109_b200.plan import PlanTrace


def _check(case):
    trace = PlanTrace.from_json(case["trace"])
    heap = replay(trace)
    gold = golden_arrays(case)
    bad = [s for s, g in gold.items() if not same_bits(heap.get(s), g)]
    assert not bad, f"{case['name']}: stores {bad} differ from the reference"


def test_bench_traces_match_reference(bench_cases):
    assert len(bench_cases) == 45
    for case in bench_cases:
        _check(case)


def test_fuzz_corpus_matches_reference(fuzz_cases):
    assert len(fuzz_cases) == 750
    for case in fuzz_cases:
        _check(case)


def test_plan_roundtrip(bench_cases):
    for case in bench_cases[:6]:
        t = PlanTrace.from_json(case["trace"])
        assert PlanTrace.from_json(t.to_json()).to_json() == t.to_json()


def test_fusion_plan_is_the_references(bench_cases):
    by = {c["name"]: c for c in bench_cases}
    rep = by["blackscholes_chain/fused"]["trace"]["meta"]["report"]
    assert rep["fused_prefixes"][-1] == 67
    assert [1, 2, 3, 6] == by["cg_csr_8x8_k2/fused"]["trace"]["meta"]["report"]["fused_prefixes"][-4:]
    assert [7, 1] == by["stencil_bands_n8_k2/fused"]["trace"]["meta"]["report"]["fused_prefixes"][-2:]


def test_spmv_csr_matches_dense_product():
    nx, ny, k = 6, 8, 2
    n = nx * ny
    dense = np.zeros((n, n))
    for p in range(k):
        rp, cl, vl = poisson_tile(nx, ny, k, p)
        t = n // k
        for i in range(t):
            for j in range(int(rp[i]), int(rp[i + 1])):
                dense[p * t + i, int(cl[j])] += vl[j]
    assert (np.diag(dense) == 4).all() and np.allclose(dense, dense.T)
    x = np.random.default_rng(0).random(n)
    y = np.concatenate([spmv_csr_rows(*poisson_tile(nx, ny, k, p), x) for p in range(k)])
    np.testing.assert_allclose(y, dense @ x, rtol=1e-14, atol=1e-14)


def test_heap_default_contents_rule():
    h = OracleHeap({0: (5, 7)}, seed=3)
    a = h.get(0).copy()
    assert a.dtype == np.float64 and a.min() >= 1 and a.max() <= 9
    h.free(0)
    assert (h.get(0) == a).all()
