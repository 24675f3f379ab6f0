"""Pins for oracle.sort (stable (key,row) order; reading R1).

Pinned by: the SPEC worked example (golden), numpy's stable argsort (a library
routine with a different algorithm), invariants (permutation, monotone, ties by
ascending row), and edge cases (empty, INT64 extremes, all-equal).
"""

import numpy as np
import pytest

import oracle
from conftest import golden

I64_MIN, I64_MAX = np.iinfo(np.int64).min, np.iinfo(np.int64).max


def test_spec_example():
    g = golden("spec_sort.json")["sort"]
    s, p = oracle.sort(g["keys"])
    assert s.tolist() == g["sorted"] and p.tolist() == g["perm"]


def test_lex_rows_by_packing():
    """Reading R12: Alg.2's sort(grps) is a lexicographic row sort; packing the
    (small, non-negative) columns into one integer reproduces SPEC.md:49."""
    g = golden("spec_sort.json")["lex_sort"]
    rows = np.array(g["rows"])
    packed = rows[:, 0] * 1000 + rows[:, 1]
    s, p = oracle.sort(packed)
    assert p.tolist() == g["perm"]
    assert rows[p].tolist() == g["sorted_rows"]


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("desc", [False, True])
def test_matches_numpy_stable(seed, desc):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 3000))
    span = [3, 100, 1 << 40][seed % 3]
    k = rng.integers(-span, span, n, dtype=np.int64)
    s, p = oracle.sort(k, descending=desc)
    ref = np.argsort(~k if desc else k, kind="stable")   # ~k reverses order without overflow
    assert np.array_equal(p, ref)
    assert np.array_equal(s, k[ref])


def test_invariants_and_edges():
    for k in [np.array([], np.int64), np.array([7]), np.full(100, 5),
              np.array([I64_MAX, I64_MIN, 0, -1, I64_MAX, I64_MIN])]:
        for desc in (False, True):
            s, p = oracle.sort(k, descending=desc)
            assert sorted(p.tolist()) == list(range(k.size))          # permutation
            assert np.array_equal(s, k[p])
            d = np.diff(s)
            assert (d <= 0).all() if desc else (d >= 0).all()          # monotone
            eq = s[1:] == s[:-1]
            assert (p[1:][eq] > p[:-1][eq]).all()                      # ties: ascending row


def test_descending_is_not_reverse():
    """Reading R1: descending keeps ties in ascending row order."""
    s, p = oracle.sort([1, 2, 1, 2], descending=True)
    assert p.tolist() == [1, 3, 0, 2]
