"""Pin the CPU oracle against the reference's own outputs (golden fixtures)."""

import numpy as np

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


def _integer_valued(arrs):
    return all(np.all(np.isfinite(a)) and np.all(a == np.round(a)) for a in arrs.values())


def test_chunked_parallel_mode_matches_reference(bench_cases, fuzz_cases, monkeypatch):
    """The full-size mode (row chunks on threads, C SPMV_CSR) reproduces the reference's heaps:
    bit-exact on integer data (every sum exact in any order), rtol 1e-12 on the real-valued CG
    plans (chunk sums are added in a different order than one np.sum)."""
    import oracle.interp as oi

    monkeypatch.setattr(oi, "_CHUNK_ELEMS", 7)  # force many chunks on the small golden stores
    calls = []
    orig = oi._interpret_chunked

    def spy(*a, **k):
        calls.append(1)
        return orig(*a, **k)

    monkeypatch.setattr(oi, "_interpret_chunked", spy)
    n_exact = n_chunked = 0
    for case in list(bench_cases) + list(fuzz_cases)[::5]:
        trace = PlanTrace.from_json(case["trace"])
        calls.clear()
        heap = replay(trace, workers=4)
        n_chunked += bool(calls)
        gold = golden_arrays(case)
        if _integer_valued(gold):
            n_exact += 1
            assert all(same_bits(heap.get(s), g) for s, g in gold.items()), case["name"]
        else:
            for s, g in gold.items():
                np.testing.assert_allclose(heap.get(s), g, rtol=1e-12, atol=1e-12 * float(np.max(np.abs(g))),
                                           err_msg=case["name"])
    assert n_exact > 100 and n_chunked > 50


def test_c_spmv_matches_numpy_restatement():
    from oracle.interp import spmv_csr_rows_c

    rng = np.random.default_rng(3)
    for nx, ny, k in ((7, 9, 1), (64, 64, 2), (33, 40, 4)):
        for p in range(k):
            rp, cl, vl = poisson_tile(nx, ny, k, p)
            vl = vl * rng.random(vl.size)
            x = rng.random(nx * ny) - 0.5
            assert same_bits(spmv_csr_rows_c(rp, cl, vl, x, 4), spmv_csr_rows(rp, cl, vl, x))
