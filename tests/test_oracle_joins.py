"""Pins for the join oracles (PK-FK: PAPER.md:55-100; m:n sort-merge: PAPER.md:286-338).

Pinned by: SPEC's worked examples and Alg. 1 trace (golden), the R4 remainder
pin, the paper's own algorithms restated literally (tests/paper_literal.py) as
an independent route, nested-loop brute force, the generator's parent-row
closed form on TPC-H-shaped data, and the size law outSize = sum_k L_k*R_k
computed with numpy's unique counts.
"""

import numpy as np
import pytest

import oracle
import paper_literal as PL
from conftest import golden


def canon(left_keys, lo, ro):
    """Sort pairs by (key, l, r) -- the canonical order (reading R6)."""
    k = np.asarray(left_keys)[lo] if len(lo) else np.array([], np.int64)
    order = np.lexsort((ro, lo, k))
    return lo[order], ro[order]


# ------------------------------------------------------------------ PK-FK

def test_pkfk_spec_example():
    g = golden("spec_pkfk.json")
    lo, ro = oracle.pkfk_join(g["build"], g["probe"])
    assert [list(x) for x in zip(lo, ro)] == g["pairs"]


def test_pkfk_duplicate_build_key():
    g = golden("spec_pkfk.json")
    with pytest.raises(oracle.OracleError) as e:
        oracle.pkfk_join(g["duplicate_build"], g["duplicate_probe"])
    assert e.value.status == oracle.ERR_DUP


def test_pkfk_macro_literal_pad_bug_and_duplicates():
    """Reading R8/R10: the literal pad min(left)-1 indexes out of range for
    probe keys below it; duplicate build keys silently drop pairs."""
    with pytest.raises(IndexError):
        PL.pkfk_join_macro([5, 6, 7], [1], pad="literal")
    lo, ro = PL.pkfk_join_macro([4, 4, 1], [4, 1], pad="safe")
    assert len(lo) == 2            # 3 true pairs, literal macro returns 2


@pytest.mark.parametrize("seed", range(40))
def test_pkfk_vs_macro_and_bruteforce(seed):
    rng = np.random.default_rng(seed)
    nb = int(rng.integers(0, 60))
    build = rng.permutation(np.arange(-50, 50))[:nb]
    probe = rng.integers(-60, 61, int(rng.integers(0, 80)))
    lo, ro = oracle.pkfk_join(build, probe)
    # ordered by probe row (reading R7)
    assert (np.diff(ro) > 0).all()
    blo, bro = oracle.nested_join(build, probe)
    assert sorted(zip(lo, ro)) == sorted(zip(blo, bro))
    if nb > 0 and probe.size > 0:
        mlo, mro = PL.pkfk_join_macro(build, probe, pad="safe")
        assert sorted(zip(lo, ro)) == sorted(zip(mlo, mro))
        # reading R7: the paper's order (probe side sorted descending, stable) is our
        # probe-row order re-sorted stably by probe key descending
        order = np.lexsort((ro, -probe[ro]))
        assert np.array_equal(lo[order], mlo) and np.array_equal(ro[order], mro)


def test_pkfk_tpch_closed_form(sf001):
    """Every lineitem row matches exactly its parent order."""
    orders, li = sf001
    lo, ro = oracle.pkfk_join(orders["o_orderkey"].numpy(), li["l_orderkey"].numpy())
    n = li["l_orderkey"].numel()
    assert np.array_equal(ro, np.arange(n))
    assert np.array_equal(lo, li["l_parent"].numpy())


def test_pkfk_tpch_filtered_build(sf001):
    """Build filter o_orderdate < 1995-03-15: pairs = {(parent[i], i): f(parent[i])}."""
    orders, li = sf001
    od = orders["o_orderdate"].numpy()
    sel = np.nonzero(od < 9204)[0]
    lo, ro = oracle.pkfk_join(orders["o_orderkey"].numpy()[sel], li["l_orderkey"].numpy())
    parent = li["l_parent"].numpy()
    keep = np.nonzero(od[parent] < 9204)[0]
    assert np.array_equal(ro, keep)
    assert np.array_equal(sel[lo], parent[keep])


# -------------------------------------------------------------- m:n join

def test_alg1_spec_trace():
    g = golden("spec_alg1_trace.json")
    lo, ro = oracle.smj_join(g["left"], g["right"])
    assert lo.tolist() == g["leftOutIdx"] and ro.tolist() == g["rightOutIdx"]
    assert oracle.smj_count(g["left"], g["right"]) == g["outSize"]
    tr = {}
    plo, pro = PL.alg1_sort_based_join(g["left"], g["right"], trace=tr)
    for k in ("leftHist", "rightHist", "histMul", "cumHistMul", "outSize", "outBucket"):
        assert tr[k] == g[k], k
    assert plo.tolist() == g["leftOutIdx"] and pro.tolist() == g["rightOutIdx"]


def test_r4_remainder_pin():
    g = golden("r4_remainder_pin.json")
    lo, ro = oracle.smj_join(g["left"], g["right"])
    assert [list(x) for x in zip(lo, ro)] == g["pairs"]
    plo, pro = PL.alg1_sort_based_join(g["left"], g["right"])
    assert [list(x) for x in zip(plo, pro)] == g["pairs"]
    with pytest.raises(IndexError):       # long-form remainder by leftHist reads past the right run
        PL.alg1_sort_based_join(g["left"], g["right"], remainder_by="left")


def test_r2_descending_variant_is_wrong():
    """Reading R2: the long form's descending sort pairs row 1 (key 1) wrongly."""
    g = golden("spec_alg1_trace.json")
    lo, _ = PL.alg1_sort_based_join(g["left"], g["right"], descending=True)
    assert lo.tolist() == [2, 2, 1, 1]
    assert lo.tolist() != g["leftOutIdx"]


@pytest.mark.parametrize("seed", range(60))
def test_smj_vs_alg1_literal_and_bruteforce(seed):
    rng = np.random.default_rng(1000 + seed)
    nl, nr = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    kmax = int(rng.integers(1, 10))
    left = rng.integers(0, kmax, nl)
    right = rng.integers(0, kmax, nr)
    lo, ro = oracle.smj_join(left, right)
    # exactly the paper's Alg. 1 (readings R2-R4), in the same order
    plo, pro = PL.alg1_sort_based_join(left, right)
    assert np.array_equal(lo, plo) and np.array_equal(ro, pro)
    # brute force, canonical order
    blo, bro = oracle.nested_join(left, right)
    clo, cro = canon(left, blo, bro)
    assert np.array_equal(lo, clo) and np.array_equal(ro, cro)
    # size law: sum over keys of L_k * R_k
    ul, cl = np.unique(left, return_counts=True)
    ur, cr = np.unique(right, return_counts=True)
    common, il, ir = np.intersect1d(ul, ur, return_indices=True)
    assert oracle.smj_count(left, right) == int((cl[il] * cr[ir]).sum()) == lo.size


@pytest.mark.parametrize("seed", range(10))
def test_smj_window_route(seed):
    rng = np.random.default_rng(2000 + seed)
    left = rng.integers(-5, 5, 300)
    right = rng.integers(-5, 5, 200)
    lo, ro = oracle.smj_join(left, right)
    n = lo.size
    for _ in range(5):
        b = int(rng.integers(0, n))
        e = int(rng.integers(b, n + 1))
        wl, wr = oracle.smj_window(left, right, b, e)
        assert np.array_equal(wl, lo[b:e]) and np.array_equal(wr, ro[b:e])


def test_smj_negative_and_wide_keys():
    """Reading R5: any int64 keys (bincount's non-negative domain is not needed)."""
    big = np.iinfo(np.int64).max
    left = np.array([big, -big - 1, 0, big, -3])
    right = np.array([-3, big, big, -big - 1])
    lo, ro = oracle.smj_join(left, right)
    blo, bro = oracle.nested_join(left, right)
    clo, cro = canon(left, blo, bro)
    assert np.array_equal(lo, clo) and np.array_equal(ro, cro)


def test_smj_empty():
    for l, r in [([], []), ([1, 2], []), ([], [3]), ([1], [2])]:
        lo, ro = oracle.smj_join(l, r)
        assert lo.size == 0 and ro.size == 0
        assert oracle.smj_count(l, r) == 0


def test_smj_zipf_uniform_size_law():
    """Config-4 shape at small scale: outSize = sum_k L_k R_k via numpy bincount."""
    from datagen import zipf_keys, uniform_keys
    left = zipf_keys(20000, 5000, seed=42).numpy()
    right = uniform_keys(20000, 5000, seed=43).numpy()
    cl = np.bincount(left, minlength=5000)
    cr = np.bincount(right, minlength=5000)
    assert oracle.smj_count(left, right) == int((cl * cr).sum())


def test_mix64_splitmix64_vectors():
    """The consumer's mix is splitmix64's output function: state += 0x9E3779B97F4A7C15,
    out = mix64(state). Published outputs for seed 0."""
    g = 0x9E3779B97F4A7C15
    assert int(oracle.mix64(g)) == 0xE220A8397B1DCDAF
    assert int(oracle.mix64((2 * g) % (1 << 64))) == 0x6E789E6AA1B965F4


def test_smj_checksum_definition():
    """The checksum of a window equals the same sums over the oracle's full join."""
    rng = np.random.default_rng(9)
    left = rng.integers(0, 30, 400)
    right = rng.integers(0, 30, 300)
    lo, ro = oracle.smj_join(left, right)
    n = lo.size
    for b, e in [(0, n), (0, 0), (7, 8), (n // 3, n - 5)]:
        h, sl, sr = oracle.smj_checksum(left, right, b, e)
        exp_h = 0
        for j in range(b, e):   # scalar route over Python ints, mod 2^64
            exp_h = (exp_h + int(oracle.mix64(int(oracle.mix64((int(lo[j]) << 32) | int(ro[j]))) ^ j))) % (1 << 64)
        assert h == exp_h
        assert sl == int(lo[b:e].sum()) % (1 << 64) and sr == int(ro[b:e].sum()) % (1 << 64)
