"""Pins for the group-by and filter oracles.

Group-by (Alg. 2): SPEC example (golden), Alg. 2 restated
literally in torch (tests/paper_literal.py), a pure-Python dict brute force,
pyarrow's hash group_by (third-party library), the Q1 closed form (exactly the
four (returnflag, linestatus) groups the generator rules allow), and exact
conservation laws with Python big integers.
Filter (Listings 1-2): the paper's predicate on SPEC's
values (golden), torch's lt/masked_select/nonzero (library), BM == SV.
"""

import math

import numpy as np
import pytest

import oracle
import paper_literal as PL
from conftest import golden
from datagen.queries import Q1_COLS, Q1_KEYS, Q1_PREDS, Q1_AGGS, Q6_COLS, Q6_PREDS, Q6_AGGS, columns


def test_groupby_spec_example():
    g = golden("spec_groupby.json")
    r = oracle.groupby_agg([g["keys"], g["values"]], [0], [("sum", [(1, 0, 1)])])
    assert r["keys"][0].tolist() == g["group_keys"] and r["results"][0] == g["sums"]


def test_unique_consecutive_semantics():
    g = golden("spec_groupby.json")["unique_consecutive"]
    r = oracle.groupby_agg([g["input"]], [0], [("count", [])])
    assert r["keys"][0].tolist() == g["unique"]
    assert np.repeat(np.arange(len(g["unique"])), r["results"][0]).tolist() == g["inverse"]
    import torch
    u, inv = torch.unique_consecutive(torch.tensor(g["input"]), return_inverse=True)
    assert u.tolist() == g["unique"] and inv.tolist() == g["inverse"]


def _brute(cols, key_idx, aggs, preds):
    ops = {"lt": lambda a, b: a < b, "le": lambda a, b: a <= b, "gt": lambda a, b: a > b,
           "ge": lambda a, b: a >= b, "eq": lambda a, b: a == b, "ne": lambda a, b: a != b}
    cols = [np.asarray(c).astype(np.int64).tolist() for c in cols]
    n = len(cols[0])
    groups = {}
    for i in range(n):
        if not all(ops[op](cols[c][i], v) for c, op, v in preds):
            continue
        key = tuple(cols[k][i] for k in key_idx)
        vals = []
        for op, fac in aggs:
            v = 1
            for c, add, sign in fac:
                v *= add + sign * cols[c][i]
            vals.append(v)
        groups.setdefault(key, []).append(vals)
    if not key_idx and not groups:
        groups[()] = []
    out = {}
    for key, rows in groups.items():
        res = []
        for a, (op, _) in enumerate(aggs):
            vs = [r[a] for r in rows]
            if op == "sum":
                res.append(sum(vs))
            elif op == "count":
                res.append(len(vs))
            elif op == "min":
                res.append(min(vs) if vs else np.iinfo(np.int64).max)
            elif op == "max":
                res.append(max(vs) if vs else np.iinfo(np.int64).min)
            else:
                res.append(float(sum(vs)) / len(vs) if vs else math.nan)
        out[key] = res
    return out


AGGS_ALL = [("sum", [(2, 0, 1)]), ("count", []), ("min", [(2, 0, 1)]), ("max", [(2, 3, -2)]),
            ("avg", [(2, 0, 1)]), ("sum", [(2, 7, -1), (1, 1, 1)])]


@pytest.mark.parametrize("seed", range(25))
def test_groupby_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 400))
    k0 = rng.integers(0, 4, n).astype(np.uint8)
    k1 = rng.integers(-3, 3, n)
    v = rng.integers(-10**12, 10**12, n)
    cols = [k0, k1, v]
    key_idx = [[0], [1], [0, 1], [1, 0], []][seed % 5]
    preds = [] if seed % 3 else [(2, "gt", -10**11)]
    r = oracle.groupby_agg(cols, key_idx, AGGS_ALL, preds)
    b = _brute(cols, key_idx, AGGS_ALL, preds)
    keys = sorted(b.keys())
    assert r["n_groups"] == len(keys)
    for gi, key in enumerate(keys):
        assert tuple(int(r["keys"][k][gi]) for k in range(len(key_idx))) == key
        for a in range(len(AGGS_ALL)):
            x, y = r["results"][a][gi], b[key][a]
            if isinstance(y, float) and math.isnan(y):
                assert math.isnan(x)
            else:
                assert x == y, (a, x, y)


@pytest.mark.parametrize("seed", range(8))
def test_groupby_vs_alg2_literal(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 500))
    k0 = rng.integers(0, 3, n)
    k1 = rng.integers(0, 5, n)
    v = rng.integers(-1000, 1000, n)
    uniq, sums, counts = PL.alg2_aggregation([k0, k1], [v])
    r = oracle.groupby_agg([k0, k1, v], [0, 1], [("sum", [(2, 0, 1)]), ("count", [])])
    assert r["keys"][0].tolist() == uniq[:, 0].tolist() and r["keys"][1].tolist() == uniq[:, 1].tolist()
    assert r["results"][0] == sums[0] and r["results"][1] == counts


def test_groupby_empty_and_global():
    r = oracle.groupby_agg([np.array([], np.int64)], [0], [("sum", [(0, 0, 1)])])
    assert r["n_groups"] == 0
    r = oracle.groupby_agg([np.array([], np.int64)], [], [("sum", [(0, 0, 1)]), ("count", []), ("min", [(0, 0, 1)]),
                                                                         ("max", [(0, 0, 1)]), ("avg", [(0, 0, 1)])])
    assert r["n_groups"] == 1
    s, c, mn, mx, av = [x[0] for x in r["results"]]
    assert (s, c, mn, mx) == (0, 0, np.iinfo(np.int64).max, np.iinfo(np.int64).min) and math.isnan(av)


def test_groupby_overflow_detected():
    big = np.array([2**62, 2**62], np.int64)
    with pytest.raises(oracle.OracleError) as e:
        oracle.groupby_agg([big], [], [("sum", [(0, 0, 1), (0, 0, 1)])])
    assert e.value.status == oracle.ERR_OVERFLOW


def test_groupby_int128_sums():
    """Reading R16: sums exceed int64 and stay exact."""
    v = np.full(10, 2**62, np.int64)
    r = oracle.groupby_agg([v], [], [("sum", [(0, 0, 1)]), ("avg", [(0, 0, 1)])])
    assert r["results"][0][0] == 10 * 2**62
    assert r["results"][1][0] == float(2**62)


def test_q1_closed_form_and_conservation(sf001):
    _, li = sf001
    cols = [c.numpy() for c in columns(li, Q1_COLS)]
    r = oracle.groupby_agg(cols, Q1_KEYS, Q1_AGGS, Q1_PREDS)
    keys = list(zip(r["keys"][0].tolist(), r["keys"][1].tolist()))
    assert keys == [(ord("A"), ord("F")), (ord("N"), ord("F")), (ord("N"), ord("O")), (ord("R"), ord("F"))]
    passing = cols[6] <= Q1_PREDS[0][2]
    assert sum(r["results"][7]) == int(passing.sum())
    qty = cols[2][passing].astype(object)
    price = cols[3][passing].astype(object)
    disc = cols[4][passing].astype(object)
    tax = cols[5][passing].astype(object)
    assert sum(r["results"][0]) == int(qty.sum())
    assert sum(r["results"][2]) == int((price * (100 - disc)).sum())
    assert sum(r["results"][3]) == int((price * (100 - disc) * (100 + tax)).sum())
    for g in range(4):     # avg = rn(sum / count) and min <= avg <= max bounds of the inputs
        assert r["results"][4][g] == float(r["results"][0][g]) / r["results"][7][g]


def test_q1_vs_pyarrow(sf001):
    """Third-party cross-check: pyarrow's hash group_by (int64 sums; valid at SF0.01)."""
    pa = pytest.importorskip("pyarrow")
    _, li = sf001
    cols = [c.numpy().astype(np.int64) for c in columns(li, Q1_COLS)]
    m = cols[6] <= Q1_PREDS[0][2]
    t = pa.table({"rf": cols[0][m], "ls": cols[1][m], "qty": cols[2][m], "price": cols[3][m],
                  "dp": cols[3][m] * (100 - cols[4][m])})
    agg = t.group_by(["rf", "ls"]).aggregate([("qty", "sum"), ("price", "sum"), ("dp", "sum"), ("qty", "count")])
    agg = agg.sort_by([("rf", "ascending"), ("ls", "ascending")]).to_pydict()
    r = oracle.groupby_agg(cols, Q1_KEYS, Q1_AGGS, Q1_PREDS)
    assert r["results"][0] == agg["qty_sum"]
    assert r["results"][1] == agg["price_sum"]
    assert r["results"][2] == agg["dp_sum"]
    assert r["results"][7] == agg["qty_count"]


# ----------------------------------------------------------------- filter

def test_filter_paper_listing_on_spec_values():
    g = golden("spec_filter.json")
    mask, sel = oracle.filter_compact([g["l_quantity"]], [(0, g["predicate"][0], g["predicate"][1])])
    assert mask.tolist() == g["mask"] and sel.tolist() == g["sel"]
    bm, vals = PL.filter_bm(g["l_quantity"], "lt", 24)
    idx, vals2 = PL.filter_sv(g["l_quantity"], "lt", 24)
    assert bm.int().tolist() == g["mask"] and idx.tolist() == g["sel"]
    assert vals.tolist() == vals2.tolist() == g["values"]


def test_q6_filter_vs_numpy_and_bm_sv(sf001):
    _, li = sf001
    cols = [c.numpy() for c in columns(li, Q6_COLS)]
    mask, sel = oracle.filter_compact(cols, Q6_PREDS)
    ref = (cols[0] >= 8766) & (cols[0] < 9131) & (cols[1] >= 5) & (cols[1] <= 7) & (cols[2] < 2400)
    assert np.array_equal(mask.astype(bool), ref)
    assert np.array_equal(sel, np.nonzero(mask)[0])                 # BM == SV
    assert 0.01 < sel.size / mask.size < 0.03                       # ~1.9% selectivity
    r = oracle.groupby_agg(cols, [], Q6_AGGS, Q6_PREDS)
    assert r["results"][0][0] == int((cols[3][ref].astype(object) * cols[1][ref].astype(object)).sum())


@pytest.mark.parametrize("op", ["lt", "le", "gt", "ge", "eq", "ne"])
def test_filter_ops_vs_torch(op):
    import torch
    rng = np.random.default_rng(7)
    c = rng.integers(-5, 5, 1000)
    mask, sel = oracle.filter_compact([c], [(0, op, 1)])
    ref = getattr(torch, op)(torch.as_tensor(c), 1).numpy()
    assert np.array_equal(mask.astype(bool), ref)
    assert np.array_equal(sel, torch.nonzero(torch.as_tensor(ref)).flatten().numpy())
