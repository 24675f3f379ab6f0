"""GPU parity: libtqp (through the C ABI) vs the CPU oracle, element by element.

Bars: indices, counts, keys and int128 sums bit-exact;
fp64 averages within 1e-12 relative (north star). Where several outputs are
correct the ABI fixes a canonical order (stable sort, probe-row order, (key, l, r)
order), so whole arrays are compared. Sizes span several tiles and ragged tails;
full-size cases (BASELINE configs[2]) use closed forms that hold at any size.
"""

import math
import os

import numpy as np
import pytest
import torch

import oracle
from conftest import golden
from datagen import random_small_keys, tpch_orders_lineitem, uniform_keys, zipf_keys
from datagen.queries import Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS, Q6_AGGS, Q6_COLS, Q6_PREDS, columns

pytestmark = pytest.mark.gpu

I64_MIN, I64_MAX = -(1 << 63), (1 << 63) - 1


@pytest.fixture(scope="module")
def T():
    import paper_2203_01877_b200 as T
    assert torch.cuda.is_available()
    return T


def cu(x, dtype=torch.int64):
    return torch.as_tensor(np.asarray(x)).to(dtype).cuda()


def npy(t):
    return t.cpu().numpy()


# ------------------------------------------------------------------- sort

def _sort_keys(kind, n, seed):
    if kind == "i64_wide":
        return random_small_keys(n, I64_MIN, I64_MAX, seed)
    if kind == "i64_narrow":
        return random_small_keys(n, 10**12, 10**12 + 5_000_000, seed)
    if kind == "i64_33bit":
        return random_small_keys(n, -(1 << 32), 1 << 32, seed)
    if kind == "i32":
        return random_small_keys(n, -(1 << 31), (1 << 31) - 1, seed, dtype=torch.int32)
    if kind == "u8":
        return random_small_keys(n, 0, 255, seed, dtype=torch.uint8)
    if kind == "dups":
        return random_small_keys(n, -3, 3, seed)
    if kind == "extremes":
        return torch.tensor([I64_MIN, I64_MAX, 0, -1], dtype=torch.int64)[random_small_keys(n, 0, 3, seed)]
    if kind == "const":
        return torch.full((n,), 42, dtype=torch.int64)
    if kind == "sorted_dups":   # already in order (the presorted shortcut), with ties
        return torch.sort(random_small_keys(n, -1000, 1000, seed)).values
    if kind == "sorted_i32_desc":   # non-increasing: identity order when sorting descending
        return torch.sort(random_small_keys(n, -(1 << 31), (1 << 31) - 1, seed, dtype=torch.int32),
                          descending=True).values
    raise ValueError(kind)


@pytest.mark.parametrize("n", [0, 1, 2, 31, 33, 3071, 3072, 3073, 4095, 4096, 4097, 100_003])
@pytest.mark.parametrize("kind", ["i64_wide", "i64_narrow", "i64_33bit", "i32", "u8", "dups", "extremes", "const",
                                  "sorted_dups", "sorted_i32_desc"])
@pytest.mark.parametrize("desc", [False, True])
def test_sort_parity(T, n, kind, desc):
    k = _sort_keys(kind, n, seed=n + 7)
    s, p = T.sort(k.cuda(), descending=desc)
    os_, op = oracle.sort(k.numpy(), descending=desc)
    assert np.array_equal(npy(p), op)
    assert np.array_equal(npy(s).astype(np.int64), os_)
    assert s.dtype == k.dtype


@pytest.mark.parametrize("dtype", [torch.int64, torch.int32])
@pytest.mark.parametrize("n", [2, 4097, 100_003, 1_000_000])
def test_sort_presorted_and_one_pair_out_of_order(T, dtype, n):
    """Sorted input takes the one-pass identity route; one adjacent pair swapped anywhere
    (first pair, across a 4,096-key tile, inside a 16-byte vector, the last pair) must not."""
    k = torch.sort(random_small_keys(n, -(1 << 30), 1 << 30, 5, dtype=dtype)).values
    cases = [k] + [k.clone() for _ in range(4)]
    for c, i in zip(cases[1:], [0, 4095, n // 2 * 2, n - 2]):
        if 0 <= i < n - 1 and c[i] != c[i + 1]:
            c[[i, i + 1]] = c[[i + 1, i]]
    for c in cases:
        for desc in (False, True):
            s, p = T.sort(c.cuda(), descending=desc)
            os_, op = oracle.sort(c.numpy(), descending=desc)
            assert np.array_equal(npy(p), op) and np.array_equal(npy(s).astype(np.int64), os_)


@pytest.mark.parametrize("kind,n", [("i64_narrow", 2_000_003), ("i64_wide", 1_000_001), ("i32", 1_500_000)])
def test_sort_parity_large(T, kind, n):
    k = _sort_keys(kind, n, seed=99)
    s, p = T.sort(k.cuda())
    _, op = oracle.sort(k.numpy())
    assert np.array_equal(npy(p), op)


# ------------------------------------------------------------------ PK-FK

def test_pkfk_spec_example(T):
    g = golden("spec_pkfk.json")
    lo, ro = T.pkfk_join(cu(g["build"]), cu(g["probe"]))
    assert [list(x) for x in zip(npy(lo), npy(ro))] == g["pairs"]


def test_pkfk_duplicate_build_key(T):
    g = golden("spec_pkfk.json")
    with pytest.raises(T.TqpError) as e:
        T.pkfk_join(cu(g["duplicate_build"]), cu(g["duplicate_probe"]))
    assert e.value.status == T.TQP_ERR_DUPLICATE_BUILD_KEY


@pytest.mark.parametrize("nb,np_,span,bd,pd", [
    (0, 0, 10, torch.int64, torch.int64), (0, 100, 10, torch.int64, torch.int64), (1, 5, 3, torch.int64, torch.int64),
    (100, 1000, 300, torch.int64, torch.int32), (5000, 100_001, 20_000, torch.int32, torch.int64),
    (2047, 2049, 4096, torch.int64, torch.int64), (300_000, 4_000_037, 1_000_000, torch.int64, torch.int64),
])
def test_pkfk_random_parity(T, nb, np_, span, bd, pd):
    rng = np.random.default_rng(nb + np_)
    build = (rng.permutation(span)[:nb] - span // 3).astype(np.int64)
    probe = rng.integers(-span // 2, span, np_).astype(np.int64)
    lo, ro = T.pkfk_join(cu(build, bd), cu(probe, pd))
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


@pytest.mark.parametrize("bits", [29, 30])
@pytest.mark.parametrize("clustered", [False, True])
def test_pkfk_fine_bucket_slot_table(T, bits, clustered):
    """Wide keys over few build rows (the SF100 shape scaled down: residual + row bits would
    need 32): the build side takes finer buckets so the slot table applies; runs of 20
    consecutive keys overflow their bucket's 8 slots (pointer route)."""
    rng = np.random.default_rng(bits + 10 * clustered)
    if clustered:
        starts = np.unique(rng.integers(0, 2**bits - 64, 5000) // 64 * 64)
        build = (starts[:, None] + np.arange(20)).ravel()
    else:
        build = np.unique(rng.integers(0, 2**bits, 110_000))
    build = rng.permutation(build).astype(np.int64)
    probe = np.concatenate([rng.choice(build, 150_000), rng.integers(-5, 2**bits + 5, 150_001)])
    probe = rng.permutation(probe).astype(np.int64)
    lo, ro = T.pkfk_join(cu(build), cu(probe))
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


@pytest.mark.parametrize("nb,np_,span", [(0, 0, 10), (1, 5, 3), (2047, 2049, 4096), (300_000, 1_000_003, 10**6)])
def test_pkfk_join_i32_outputs(T, nb, np_, span):
    """tqp_pkfk_join_i32: the oracle's pairs, written as int32."""
    rng = np.random.default_rng(nb + np_ + 7)
    build = (rng.permutation(span)[:nb] - span // 3).astype(np.int64)
    probe = rng.integers(-span // 2, span, np_).astype(np.int64)
    lo, ro = T.pkfk_join(cu(build), cu(probe), index_dtype=torch.int32)
    assert lo.dtype == torch.int32 and ro.dtype == torch.int32
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo).astype(np.int64), olo) and np.array_equal(npy(ro).astype(np.int64), oro)


@pytest.mark.parametrize("nb,np_,span,pd", [(0, 100, 10, torch.int64), (1, 5, 3, torch.int64), (50, 3000, 40, torch.int32),
                                             (5000, 100_001, 20_000, torch.int64), (300_000, 1_000_003, 10**6, torch.int64)])
def test_pkfk_join_paper_order(T, nb, np_, span, pd):
    """Reading R7: the paper's order = the oracle's pairs re-sorted stably by probe key
    descending (ties: ascending probe row)."""
    rng = np.random.default_rng(nb + np_ + 11)
    build = (rng.permutation(span)[:nb] - span // 3).astype(np.int64)
    probe = rng.integers(-span // 2, span, np_).astype(np.int64)
    lo, ro = T.pkfk_join_paper_order(cu(build), cu(probe, pd))
    olo, oro = oracle.pkfk_join(build, probe)
    order = np.lexsort((oro, -probe[oro]))
    assert np.array_equal(npy(lo), olo[order]) and np.array_equal(npy(ro), oro[order])


def test_pkfk_join_paper_order_extremes(T):
    build = np.array([I64_MAX, I64_MIN, 0, -1, 5], np.int64)
    probe = np.array([5, I64_MIN, I64_MAX, 7, 0, I64_MIN, -1, 5, I64_MAX], np.int64)
    lo, ro = T.pkfk_join_paper_order(cu(build), cu(probe))
    olo, oro = oracle.pkfk_join(build, probe)
    order = sorted(range(olo.size), key=lambda j: (-int(probe[oro[j]]), int(oro[j])))
    assert npy(lo).tolist() == olo[order].tolist() and npy(ro).tolist() == oro[order].tolist()


@pytest.mark.parametrize("nb,np_,span", [(0, 100, 10), (1, 5, 3), (5000, 100_001, 20_000), (300_000, 1_000_003, 10**6)])
def test_pkfk_hash_ablation_parity(T, nb, np_, span):
    """The hash-join ablation returns exactly the sort-based join's output (and the oracle's)."""
    rng = np.random.default_rng(nb + np_ + 1)
    build = (rng.permutation(span)[:nb] - span // 3).astype(np.int64)
    probe = rng.integers(-span // 2, span, np_).astype(np.int64)
    lo, ro = T.pkfk_join_hash(cu(build), cu(probe))
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    with pytest.raises(T.TqpError) as e:
        T.pkfk_join_hash(cu(np.array([7, 3, 7])), cu(probe[:10]))
    assert e.value.status == T.TQP_ERR_DUPLICATE_BUILD_KEY


def test_pkfk_wide_and_extreme_keys(T):
    build = np.array([I64_MIN, I64_MAX, 0, -1, 1 << 40, -(1 << 50)], np.int64)
    probe = np.array([I64_MAX, 5, I64_MIN, -1, 1 << 40, 0, I64_MAX, -(1 << 50) + 1], np.int64)
    lo, ro = T.pkfk_join(cu(build), cu(probe))
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


def test_pkfk_tpch_sf1_parity_and_closed_form(T):
    orders, li = tpch_orders_lineitem(1.0, seed=42, device="cuda")
    lo, ro = T.pkfk_join(orders["o_orderkey"], li["l_orderkey"])
    n = li["l_orderkey"].numel()
    assert torch.equal(ro, torch.arange(n, device="cuda"))
    assert torch.equal(lo, li["l_parent"])
    olo, oro = oracle.pkfk_join(npy(orders["o_orderkey"]), npy(li["l_orderkey"]))
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


def test_pkfk_tpch_filtered_build(T):
    orders, li = tpch_orders_lineitem(0.01, seed=42, device="cuda")
    _, sel = T.filter_compact([orders["o_orderdate"]], [(0, "lt", 9204)], mask=False)
    bk = orders["o_orderkey"][sel]
    lo, ro = T.pkfk_join(bk, li["l_orderkey"])
    olo, oro = oracle.pkfk_join(npy(bk), npy(li["l_orderkey"]))
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


@pytest.mark.parametrize("kind", ["dense", "sparse", "i32_negative", "block_edges", "one_key"])
def test_pkfk_presorted_build_rank_bitmap(T, kind):
    """Build sides already in key order take the rank-bitmap route (one 32-byte block of a
    rank + 224 presence bits per probe): dense and sparse domains, negative i32 keys, keys
    on 224-bit block edges; probe keys below, inside and above the domain."""
    rng = np.random.default_rng(7)
    if kind == "dense":
        build = np.arange(-50_000, 250_000, dtype=np.int64)
    elif kind == "sparse":
        build = np.unique(rng.integers(0, 6_000_000, 400_000))
    elif kind == "i32_negative":
        build = np.unique(rng.integers(-(1 << 31), -(1 << 31) + 3_000_000, 200_000))
    elif kind == "block_edges":
        e = np.arange(1, 3000, dtype=np.int64) * 224
        build = np.unique(np.concatenate([e - 1, e, e + 1, e + 31, e + 32, e + 95, e + 96]))
    else:
        build = np.array([123456789], dtype=np.int64)
    dt = torch.int32 if kind == "i32_negative" else torch.int64
    lo_, hi_ = int(build.min()), int(build.max())
    probe = np.concatenate([rng.choice(build, 300_000), rng.integers(lo_ - 300, hi_ + 300, 300_001)])
    if dt == torch.int32:
        probe = np.clip(probe, -(1 << 31), (1 << 31) - 1)
    probe = rng.permutation(probe).astype(np.int64)
    lo, ro = T.pkfk_join(cu(build, dt), cu(probe, dt))
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    left, mask = T.pkfk_outer(cu(build, dt), cu(probe, dt), return_mask=True)   # probe-side outer join
    want = np.full(probe.size, -1, np.int64)
    want[oro] = olo
    assert np.array_equal(npy(left), want) and np.array_equal(npy(mask).astype(bool), want >= 0)
    dups = np.sort(np.concatenate([build, build[::3]]))   # semi / anti: duplicates allowed
    for anti in (False, True):
        sel = T.pkfk_semi(cu(dups, dt), cu(probe, dt), anti=anti)
        member = np.isin(probe, build)
        assert np.array_equal(npy(sel), np.nonzero(~member if anti else member)[0])
    if build.size > 1:   # a duplicate in a presorted build side is still an error
        with pytest.raises(T.TqpError) as e:
            T.pkfk_join(cu(np.insert(build, 1, build[0]), dt), cu(probe[:10], dt))
        assert e.value.status == T.TQP_ERR_DUPLICATE_BUILD_KEY


@pytest.mark.parametrize("slice_mb", ["0.004", "0.05"])
def test_pkfk_multipass_probe(T, slice_mb):
    """The multi-pass probe (build sides much larger than L2, e.g. SF100) run at small sizes
    by shrinking its slice: several passes, ragged tiles, i32 keys, a sparse key domain."""
    import subprocess
    import sys
    env = dict(os.environ, TQP_PROBE_SLICE_MB=slice_mb)
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_pkfk_multipass_child.py")
    r = subprocess.run([sys.executable, child], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


def test_pkfk_sf10_full_size_closed_form(T):
    """BASELINE configs[2] at full size (15M x 60M), in bench.py's launch configuration:
    every lineitem row matches exactly its parent order (generator closed form)."""
    orders, li = tpch_orders_lineitem(10.0, seed=42, device="cuda")
    lo, ro = T.pkfk_join(orders["o_orderkey"], li["l_orderkey"])
    assert lo.numel() == li["l_orderkey"].numel()
    assert torch.equal(ro, torch.arange(lo.numel(), device="cuda"))
    assert torch.equal(lo, li["l_parent"])
    # sampled rows against the oracle's definition, one by one
    idx = torch.randint(0, lo.numel(), (64,), generator=torch.Generator().manual_seed(1)).tolist()
    ok = npy(orders["o_orderkey"])
    for i in idx:
        key = int(li["l_orderkey"][i])
        blo, _ = oracle.pkfk_join(ok, np.array([key]))
        assert int(lo[i]) == int(blo[0])


def test_smj_sf10_full_size_closed_form(T):
    """The bench's SMJ (orders x lineitem at SF10, full size, same calls as bench.py): the
    pairs are (parent[r], r) in (key, l, r) order; order keys ascend with the order row, so
    that is lineitem rows stably sorted by parent (torch: a library route). Sampled pair
    windows against the oracle's per-offset definition."""
    orders, li = tpch_orders_lineitem(10.0, seed=42, device="cuda")
    ok, lk = orders["o_orderkey"], li["l_orderkey"]
    plan = T.smj_prepare(ok, lk)
    assert plan.size == lk.numel()
    lo, ro = plan.expand(0, plan.size)
    want_ro = torch.sort(li["l_parent"], stable=True).indices
    assert torch.equal(ro, want_ro)
    assert torch.equal(lo, li["l_parent"][want_ro])
    plan.release()
    # windows: the oracle on the keys of a slice of orders (its pairs are a contiguous
    # range of the full output, shifted by the lineitems of the preceding orders)
    o0, o1 = 7_000_000, 7_000_400
    sel = ((lk >= ok[o0]) & (lk <= ok[o1 - 1])).nonzero().flatten()
    olo, oro = oracle.smj_join(npy(ok[o0:o1]), npy(lk[sel]))
    start = int((lk < ok[o0]).sum())
    assert np.array_equal(npy(lo[start:start + olo.size]) - o0, olo)
    assert np.array_equal(npy(ro[start:start + oro.size]), npy(sel)[oro])


@pytest.mark.parametrize("anti", [False, True])
def test_pkfk_semi_anti(T, anti):
    rng = np.random.default_rng(5)
    build = rng.integers(0, 5000, 3000)      # duplicates allowed for semi/anti
    probe = rng.integers(-100, 6000, 50_001)
    sel, mask = T.pkfk_semi(cu(build), cu(probe), anti=anti, return_mask=True)
    member = np.isin(probe, build)
    assert np.array_equal(npy(mask).astype(bool), member)
    want = np.nonzero(~member if anti else member)[0]
    assert np.array_equal(npy(sel), want)
    # cross-check against the oracle join on the de-duplicated build side
    _, r = oracle.pkfk_join(np.unique(build), probe)
    assert np.array_equal(np.nonzero(member)[0], r)


@pytest.mark.parametrize("indices", [True, False])
def test_pkfk_join_payload(T, indices):
    """Payload columns gathered into the join output equal the columns gathered by the
    oracle's index pairs (u8 / i32 / i64 payloads on both sides)."""
    orders, li = tpch_orders_lineitem(0.05, seed=42, device="cuda")
    ok, lk = orders["o_orderkey"], li["l_orderkey"]
    keep = torch.arange(ok.numel(), device="cuda") % 3 != 0           # a third of the orders unmatched
    bk = ok[keep]
    bpay = [orders["o_orderdate"][keep], bk * 7 - 3]
    ppay = [li["l_returnflag"], li["l_shipdate"], li["l_extendedprice"]]
    bo, po, idx = T.pkfk_join_payload(bk, lk, bpay, ppay, indices=indices)
    olo, oro = oracle.pkfk_join(npy(bk), npy(lk))
    for got, col in zip(bo, bpay):
        assert np.array_equal(npy(got), npy(col)[olo])
    for got, col in zip(po, ppay):
        assert np.array_equal(npy(got), npy(col)[oro])
    if indices:
        assert np.array_equal(npy(idx[0]), olo) and np.array_equal(npy(idx[1]), oro)


@pytest.mark.parametrize("nb,np_,span", [(0, 1000, 50), (1, 5, 3), (3000, 50_001, 6000), (300_000, 1_000_003, 10**6)])
def test_pkfk_outer(T, nb, np_, span):
    """Probe-side outer join: every probe row, its build row or -1 (oracle pairs fill the rest)."""
    rng = np.random.default_rng(nb + 7)
    build = (rng.permutation(span)[:nb] - span // 4).astype(np.int64)
    probe = rng.integers(-span // 2, span, np_).astype(np.int64)
    left, mask = T.pkfk_outer(cu(build), cu(probe), return_mask=True)
    olo, oro = oracle.pkfk_join(build, probe)
    want = np.full(np_, -1, np.int64)
    want[oro] = olo
    assert np.array_equal(npy(left), want)
    assert np.array_equal(npy(mask).astype(bool), want >= 0)


@pytest.mark.parametrize("presorted", [True, False])
def test_pkfk_outer_duplicate_build_keys(T, presorted):
    """Outer join over a build side with duplicate keys (not an error for the outer join):
    each probe row takes a build row with its key, or -1. A presorted build side is the
    rank-bitmap route, whose rank + popcount row would be wrong with duplicates (ADVICE r01:
    [5,5,6] probed with 6 gave row 1), so it must be rebuilt without it."""
    rng = np.random.default_rng(11)
    build = rng.integers(0, 50_000, 200_003).astype(np.int64)
    build[:3] = [5, 5, 6]
    if presorted:
        build = np.sort(build)
    probe = rng.integers(-100, 51_000, 300_001).astype(np.int64)
    probe[:2] = [6, 5]
    left, mask = T.pkfk_outer(cu(build), cu(probe), return_mask=True)
    left = npy(left)
    members = set(build.tolist())
    want_match = np.array([p in members for p in probe.tolist()])
    assert np.array_equal(npy(mask).astype(bool), want_match)
    assert np.array_equal(left >= 0, want_match)
    assert np.array_equal(build[left[want_match]], probe[want_match])   # a build row with the probe key


def test_pkfk_semi_empty_build(T):
    sel = T.pkfk_semi(cu(np.array([], np.int64)), cu(np.arange(10)), anti=True)
    assert npy(sel).tolist() == list(range(10))
    assert T.pkfk_semi(cu(np.array([], np.int64)), cu(np.arange(10))).numel() == 0


# -------------------------------------------------------------------- SMJ

def test_smj_alg1_trace(T):
    g = golden("spec_alg1_trace.json")
    plan = T.smj_prepare(cu(g["left"]), cu(g["right"]))
    assert plan.size == g["outSize"]
    lo, ro = plan.expand(0, plan.size)
    assert npy(lo).tolist() == g["leftOutIdx"] and npy(ro).tolist() == g["rightOutIdx"]


def test_smj_r4_pin(T):
    g = golden("r4_remainder_pin.json")
    lo, ro = T.smj_join(cu(g["left"]), cu(g["right"]))
    assert [list(x) for x in zip(npy(lo), npy(ro))] == g["pairs"]


@pytest.mark.parametrize("seed", range(12))
def test_smj_random_parity(T, seed):
    rng = np.random.default_rng(seed)
    nl = int(rng.integers(0, 6000))
    nr = int(rng.integers(0, 6000))
    kmax = int(rng.choice([3, 50, 2000, 10**6]))
    left = rng.integers(-kmax, kmax, nl)
    right = rng.integers(-kmax, kmax, nr)
    lo, ro = T.smj_join(cu(left), cu(right))
    olo, oro = oracle.smj_join(left, right)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


def test_smj_dtypes_and_extremes(T):
    left = np.array([I64_MAX, I64_MIN, 0, I64_MAX, -3, 7], np.int64)
    right = np.array([-3, I64_MAX, I64_MAX, I64_MIN, 7, 7], np.int64)
    lo, ro = T.smj_join(cu(left), cu(right))
    olo, oro = oracle.smj_join(left, right)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    l32 = np.array([1, 2, 2, 300], np.int64)
    lo, ro = T.smj_join(cu(l32, torch.int32), cu(np.array([2, 300, 2]), torch.int64))
    olo, oro = oracle.smj_join(l32, [2, 300, 2])
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


@pytest.mark.parametrize("case", ["same_hi", "diff_hi", "wide_left", "wide_right", "negative", "const_sides"])
def test_smj_key_domains(T, case):
    """The join compares sorted keys in a common domain: 32-bit unique keys when both
    sides vary only in the same low word, 64-bit otherwise (mixed widths, different high
    words, one-key sides)."""
    rng = np.random.default_rng(len(case))
    n = 30_011
    base = {"same_hi": (5 << 32, 5 << 32), "diff_hi": (5 << 32, 6 << 32), "wide_left": (0, 0),
            "wide_right": (0, 0), "negative": (-(1 << 33), -(1 << 33)), "const_sides": (7, 7)}[case]
    left = base[0] + rng.integers(0, 5000, n)
    right = base[1] + rng.integers(0, 5000, n)
    if case == "wide_left":
        left[::97] = rng.integers(1 << 40, 1 << 41, left[::97].size)
    if case == "wide_right":
        right[::89] = -rng.integers(1 << 40, 1 << 41, right[::89].size)
    if case == "diff_hi":   # some keys shared across the two high words
        right[::50] = left[::50][: right[::50].size]
    if case == "const_sides":   # one distinct key on the left (trivial sort), ~45K pairs
        left = np.full(300, 7, np.int64)
        right = right[:301].copy()
        right[::2] = 7
    lo, ro = T.smj_join(cu(left), cu(right))
    olo, oro = oracle.smj_join(left, right)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


def test_smj_zipf_uniform_parity(T):
    """Config-4 shape (Zipf(s=1) left x uniform right) at 400K x 400K."""
    left = zipf_keys(400_000, 400_000, seed=42, device="cuda")
    right = uniform_keys(400_000, 400_000, seed=43, device="cuda")
    plan = T.smj_prepare(left, right)
    assert plan.size == oracle.smj_count(npy(left), npy(right))
    lo, ro = plan.expand(0, plan.size)
    olo, oro = oracle.smj_join(npy(left), npy(right))
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    # windows, including ragged ones crossing the heavy key's bucket
    rng = np.random.default_rng(3)
    for _ in range(4):
        b = int(rng.integers(0, plan.size))
        e = int(min(plan.size, b + rng.integers(1, 50_000)))
        wl, wr = plan.expand(b, e)
        assert np.array_equal(npy(wl), olo[b:e]) and np.array_equal(npy(wr), oro[b:e])
    plan.release()


def test_smj_expand_i32_outputs(T):
    """tqp_smj_expand_i32: full expansion and ragged / unaligned windows match the oracle."""
    left = zipf_keys(100_000, 100_000, seed=44, device="cuda")
    right = uniform_keys(100_000, 100_000, seed=45, device="cuda")
    plan = T.smj_prepare(left, right)
    olo, oro = oracle.smj_join(npy(left), npy(right))
    lo, ro = plan.expand(0, plan.size, index_dtype=torch.int32)
    assert lo.dtype == torch.int32
    assert np.array_equal(npy(lo).astype(np.int64), olo) and np.array_equal(npy(ro).astype(np.int64), oro)
    rng = np.random.default_rng(5)
    buf_l = torch.empty(60_001, dtype=torch.int32, device="cuda")
    buf_r = torch.empty(60_001, dtype=torch.int32, device="cuda")
    for _ in range(4):
        b = int(rng.integers(0, plan.size))
        e = int(min(plan.size, b + rng.integers(1, 50_000)))
        off = int(rng.integers(0, 3))   # unaligned output start: scalar store path
        plan.expand(b, e, out=(buf_l[off:], buf_r[off:]))
        assert np.array_equal(npy(buf_l[off:off + e - b]).astype(np.int64), olo[b:e])
        assert np.array_equal(npy(buf_r[off:off + e - b]).astype(np.int64), oro[b:e])
    with pytest.raises(ValueError):
        plan.expand(0, 10, out=(buf_l, buf_r.to(torch.int64)))
    plan.release()


def test_smj_expand_checksum(T):
    """The fused consumer (no materialisation) equals the oracle's checksum on full and
    ragged windows, including windows crossing the heavy Zipf key."""
    left = zipf_keys(60_000, 60_000, seed=46, device="cuda")
    right = uniform_keys(60_000, 60_000, seed=47, device="cuda")
    plan = T.smj_prepare(left, right)
    L, R = npy(left), npy(right)
    rng = np.random.default_rng(6)
    wins = [(0, plan.size), (0, 0), (5, 6), (plan.size - 1, plan.size)]
    for _ in range(4):
        b = int(rng.integers(0, plan.size))
        wins.append((b, int(min(plan.size, b + rng.integers(1, 40_000)))))
    for b, e in wins:
        assert plan.checksum(b, e) == oracle.smj_checksum(L, R, b, e), (b, e)
    plan.release()


def test_smj_checksum_both_zipf_windows(T):
    """Config-4 as stated (both Zipf, outSize not materialisable at full size): windowed
    checksums against the oracle's per-offset route."""
    left = zipf_keys(200_000, 10**6, seed=42, device="cuda")
    right = zipf_keys(200_000, 10**6, seed=43, stream=101, device="cuda")
    plan = T.smj_prepare(left, right)
    rng = np.random.default_rng(8)
    for b in [0] + [int(x) for x in rng.integers(0, plan.size - 100_000, 3)]:
        assert plan.checksum(b, b + 100_000) == oracle.smj_checksum(npy(left), npy(right), b, b + 100_000)
    plan.release()


def test_smj_coarse_tile_table(T):
    """outSize ~9.6e9 from two heavy keys (the coarse tile-bucket table path): windows
    crossing the heavy-heavy and heavy-light boundaries, materialised and checksummed."""
    left = np.concatenate([np.full(60_000, 1), np.full(60_000, 2), np.arange(3, 1003)]).astype(np.int64)
    right = np.concatenate([np.arange(3, 1003), np.full(80_000, 2), np.full(80_000, 1)]).astype(np.int64)
    rng = np.random.default_rng(10)
    left, right = rng.permutation(left), rng.permutation(right)
    plan = T.smj_prepare(cu(left), cu(right))
    assert plan.size == oracle.smj_count(left, right) == 2 * 60_000 * 80_000 + 1000
    h = 60_000 * 80_000
    wins = [(0, 5000), (h - 3000, h + 3000), (2 * h - 10, plan.size), (plan.size - 7, plan.size)]
    wins += [(int(b), int(b) + 20_000) for b in rng.integers(0, plan.size - 20_000, 3)]
    for b, e in wins:
        lo, ro = plan.expand(b, e)
        olo, oro = oracle.smj_window(left, right, b, e)
        assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro), (b, e)
        assert plan.checksum(b, e) == oracle.smj_checksum(left, right, b, e), (b, e)
    plan.release()


def _dense_ids(a_cols, b_cols):
    """Tuple -> id in lexicographic tuple order over both sides (numpy unique on rows)."""
    ta = np.stack([np.asarray(c, np.int64) for c in a_cols], axis=1)
    tb = np.stack([np.asarray(c, np.int64) for c in b_cols], axis=1)
    _, inv = np.unique(np.concatenate([ta, tb]), axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    return inv[:len(ta)], inv[len(ta):]


def test_pack_keys_composite_joins(T):
    """Composite keys (i32, u8, i64 with negatives): PK-FK and SMJ on the packed keys equal
    the oracle's joins on the tuples' dense ids (independent densification)."""
    rng = np.random.default_rng(12)
    nb, np_ = 3000, 20_011
    # unique build tuples over a small domain
    dom = np.array([(a, b, c) for a in range(-20, 20) for b in range(0, 256, 37) for c in (-(1 << 40), 0, 77)])
    bt = dom[rng.permutation(len(dom))[:nb]]
    pt = dom[rng.integers(0, len(dom), np_)]
    pt[::13, 2] = 5   # tuples absent from the build side
    bcols = [cu(bt[:, 0], torch.int32), cu(bt[:, 1], torch.uint8), cu(bt[:, 2])]
    pcols = [cu(pt[:, 0], torch.int32), cu(pt[:, 1], torch.uint8), cu(pt[:, 2])]
    kb, kp, bits = T.pack_keys(bcols, pcols)
    assert bits <= 63
    ib, ip = _dense_ids([bt[:, 0], bt[:, 1], bt[:, 2]], [pt[:, 0], pt[:, 1], pt[:, 2]])
    lo, ro = T.pkfk_join(kb, kp)
    olo, oro = oracle.pkfk_join(ib, ip)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    # m:n join on composite keys: same pairs in the same (key, l, r) order
    lt, rt = pt[:5000], pt[5000:9000]
    kl, kr, _ = T.pack_keys([cu(lt[:, 0], torch.int32), cu(lt[:, 1], torch.uint8), cu(lt[:, 2])],
                            [cu(rt[:, 0], torch.int32), cu(rt[:, 1], torch.uint8), cu(rt[:, 2])])
    il, ir = _dense_ids([lt[:, 0], lt[:, 1], lt[:, 2]], [rt[:, 0], rt[:, 1], rt[:, 2]])
    lo, ro = T.smj_join(kl, kr)
    olo, oro = oracle.smj_join(il, ir)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


def test_pack_keys_edges(T):
    one = cu(np.array([5, 5, 5]))
    ka, kb, bits = T.pack_keys([one], [cu(np.array([5]))])
    assert bits == 0 and npy(ka).tolist() == [0, 0, 0] and npy(kb).tolist() == [0]
    ka, kb, bits = T.pack_keys([cu(np.array([3, 1, 2]))])   # one side only
    assert kb is None and npy(ka).tolist() == [2, 0, 1] and bits == 2
    wide = cu(np.array([I64_MIN, I64_MAX]))
    with pytest.raises(T.TqpError):
        T.pack_keys([wide, cu(np.array([0, 1]))])   # 64 + 1 bits


def test_smj_both_zipf_windows(T):
    """Config-4 as stated (both sides Zipf): outSize exact; windows by the oracle's per-offset route."""
    left = zipf_keys(200_000, 10**6, seed=42, device="cuda")
    right = zipf_keys(200_000, 10**6, seed=43, stream=101, device="cuda")
    plan = T.smj_prepare(left, right)
    assert plan.size == oracle.smj_count(npy(left), npy(right))
    rng = np.random.default_rng(4)
    for b in [0] + [int(x) for x in rng.integers(0, plan.size - 5000, 3)]:
        wl, wr = plan.expand(b, b + 5000)
        olo, oro = oracle.smj_window(npy(left), npy(right), b, b + 5000)
        assert np.array_equal(npy(wl), olo) and np.array_equal(npy(wr), oro)
    plan.release()


def test_smj_empty(T):
    for l, r in [([], []), ([1, 2], []), ([], [3]), ([1], [2])]:
        lo, ro = T.smj_join(cu(np.array(l, np.int64)), cu(np.array(r, np.int64)))
        assert lo.numel() == 0 and ro.numel() == 0


# ----------------------------------------------------------------- filter

def test_filter_spec_listing(T):
    g = golden("spec_filter.json")
    mask, sel = T.filter_compact([cu(g["l_quantity"])], [(0, "lt", 24)])
    assert npy(mask).tolist() == g["mask"] and npy(sel).tolist() == g["sel"]


@pytest.mark.parametrize("n", [0, 1, 2047, 2048, 2049, 1_000_003])
def test_filter_random_parity(T, n):
    rng = np.random.default_rng(n)
    a = rng.integers(-50, 50, n)
    b = rng.integers(0, 256, n).astype(np.uint8)
    c = rng.integers(-10**6, 10**6, n).astype(np.int32)
    cols = [a, b, c]
    preds = [(0, "ge", -20), (1, "ne", 7), (2, "lt", 500_000), (0, "le", 45)]
    mask, sel = T.filter_compact([cu(a), cu(b, torch.uint8), cu(c, torch.int32)], preds)
    om, os_ = oracle.filter_compact(cols, preds)
    assert np.array_equal(npy(mask), om) and np.array_equal(npy(sel), os_)


@pytest.mark.parametrize("preds", [[], [(0, "lt", -100)], [(0, "ge", -100)]])
def test_filter_all_or_none(T, preds):
    a = np.arange(-50, 50)
    mask, sel = T.filter_compact([cu(a)], preds)
    om, os_ = oracle.filter_compact([a], preds)
    assert np.array_equal(npy(mask), om) and np.array_equal(npy(sel), os_)


I64_MIN, I64_MAX = -(1 << 63), (1 << 63) - 1
FOLD_CASES = [   # the library folds each column's predicates into one interval (common.cuh make_terms)
    [(0, "gt", 10), (0, "lt", 5)],                          # contradiction: nothing passes
    [(0, "lt", I64_MIN)], [(0, "gt", I64_MAX)],             # empty at the int64 ends
    [(0, "le", I64_MAX), (0, "ge", I64_MIN)],               # the whole domain
    [(1, "eq", 300)], [(1, "ne", 300)], [(1, "lt", 0)], [(1, "ge", -5)],   # u8 beyond its domain
    [(2, "gt", 1 << 40)], [(2, "ge", -(1 << 40)), (2, "le", 1 << 40)],     # i32 beyond its domain
    [(1, "ne", 0), (1, "ne", 255), (1, "gt", 3), (1, "le", 200), (1, "ne", 100)],
    [(0, "eq", 7), (0, "ge", 7), (0, "le", 7), (2, "ne", 0)],
    [(0, "ge", -20), (0, "le", 45), (0, "gt", -30), (0, "lt", 40), (2, "lt", 0), (2, "gt", -500_000)],
    [(2, "eq", 12345), (2, "ne", 12345)],
]


def fold_inputs(n, seed=5):
    rng = np.random.default_rng(seed)
    a = rng.integers(-50, 50, n)
    a[:4] = [I64_MIN, I64_MAX, 7, -7]
    b = rng.integers(0, 256, n).astype(np.uint8)
    c = rng.integers(-10**6, 10**6, n).astype(np.int32)
    c[:3] = [np.iinfo(np.int32).min, np.iinfo(np.int32).max, 12345]
    return [a, b, c]


@pytest.mark.parametrize("k", range(len(FOLD_CASES)))
def test_filter_predicate_folding(T, k):
    cols = fold_inputs(100_003)
    preds = FOLD_CASES[k]
    mask, sel = T.filter_compact([cu(cols[0]), cu(cols[1], torch.uint8), cu(cols[2], torch.int32)], preds)
    om, os_ = oracle.filter_compact(cols, preds)
    assert np.array_equal(npy(mask), om) and np.array_equal(npy(sel), os_)


@pytest.mark.parametrize("k", range(len(FOLD_CASES)))
def test_groupby_predicate_folding(T, k):
    """Both group-by tile paths (keyed: strided rows; no key: vector rows + pass lists)."""
    cols = fold_inputs(50_001)
    g = (cols[0] & 3).astype(np.int64)
    dcols = [cu(cols[0]), cu(cols[1], torch.uint8), cu(cols[2], torch.int32), cu(g)]
    hcols = cols + [g]
    aggs = [("sum", [(2, 0, 1)]), ("count", []), ("max", [(1, 0, 1)]), ("min", [(2, 1, -1)])]
    for keys in ([3], []):
        got = T.groupby_agg(dcols, keys, aggs, FOLD_CASES[k])
        want = oracle.groupby_agg(hcols, keys, aggs, FOLD_CASES[k])
        check_groupby(T, got, want, aggs)


def test_filter_unaligned_columns(T):
    """Columns starting 8 bytes into an allocation take the scalar loads."""
    base = torch.randint(-100, 100, (300_001,), dtype=torch.int64, device="cuda")
    x = base[1:]
    assert x.data_ptr() % 16 != 0
    preds = [(0, "ge", -20), (0, "lt", 60)]
    mask, sel = T.filter_compact([x], preds)
    om, os_ = oracle.filter_compact([npy(x)], preds)
    assert np.array_equal(npy(mask), om) and np.array_equal(npy(sel), os_)


def test_filter_q6_sf1(T):
    _, li = tpch_orders_lineitem(1.0, seed=42, device="cuda")
    cols = columns(li, Q6_COLS)
    mask, sel = T.filter_compact(cols, Q6_PREDS)
    om, os_ = oracle.filter_compact([npy(c) for c in cols], Q6_PREDS)
    assert np.array_equal(npy(mask), om) and np.array_equal(npy(sel), os_)


# ---------------------------------------------------------------- group-by

def check_groupby(T, got, want, aggs):
    assert got["n_groups"] == want["n_groups"]
    for k in range(len(got["keys"])):
        assert np.array_equal(npy(got["keys"][k]).astype(np.int64), want["keys"][k])
    for a, (op, _) in enumerate(aggs):
        w = want["results"][a]
        if op == "sum":
            assert T.int128_to_ints(got["results"][a]) == w
        elif op == "avg":
            g = npy(got["results"][a]).tolist()
            for x, y in zip(g, w):
                if math.isnan(y):
                    assert math.isnan(x)
                else:
                    assert abs(x - y) <= 1e-12 * max(abs(y), 1e-300)
        else:
            assert npy(got["results"][a]).tolist() == w


def test_groupby_spec_example(T):
    g = golden("spec_groupby.json")
    aggs = [("sum", [(1, 0, 1)])]
    got = T.groupby_agg([cu(g["keys"]), cu(g["values"])], [0], aggs)
    assert npy(got["keys"][0]).tolist() == g["group_keys"]
    assert T.int128_to_ints(got["results"][0]) == g["sums"]


@pytest.fixture(params=["jit", "generic"])
def dense_kernel(request, monkeypatch):
    """The dense group-by kernel compiled for the plan (jit.cu; TQP_JIT_MIN_ROWS=0 so every
    size uses it) or the generic one (TQP_JIT=0): both must give the oracle's result."""
    if request.param == "jit":
        monkeypatch.setenv("TQP_JIT_MIN_ROWS", "0")
    else:
        monkeypatch.setenv("TQP_JIT", "0")
    return request.param


@pytest.mark.parametrize("sf", [0.01, 1.0])
def test_groupby_q1_parity(T, sf, dense_kernel):
    _, li = tpch_orders_lineitem(sf, seed=42, device="cuda")
    cols = columns(li, Q1_COLS)
    jit0 = T.jit_counters()
    got = T.groupby_agg(cols, Q1_KEYS, Q1_AGGS, Q1_PREDS)
    want = oracle.groupby_agg([npy(c) for c in cols], Q1_KEYS, Q1_AGGS, Q1_PREDS)
    check_groupby(T, got, want, Q1_AGGS)
    if dense_kernel == "jit":   # Q1's four (returnflag, linestatus) groups: the compiled kernel
        assert T.jit_counters()["launches"] > jit0["launches"]


def test_groupby_q6_fused_sum(T):
    _, li = tpch_orders_lineitem(1.0, seed=42, device="cuda")
    cols = columns(li, Q6_COLS)
    got = T.groupby_agg(cols, [], Q6_AGGS, Q6_PREDS)
    want = oracle.groupby_agg([npy(c) for c in cols], [], Q6_AGGS, Q6_PREDS)
    check_groupby(T, got, want, Q6_AGGS)


AGGS_ALL = [("sum", [(2, 0, 1)]), ("count", []), ("min", [(2, 0, 1)]), ("max", [(2, 3, -1)]),
            ("avg", [(2, 0, 1)]), ("sum", [(2, 7, -1), (1, 1, 1)]), ("min", [(3, 0, 1)]), ("max", [(3, 5, 1)])]


@pytest.mark.parametrize("seed", range(10))
def test_groupby_random_parity(T, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([0, 1, 2047, 2048, 2049, 50_000, 300_001]))
    card = int(rng.choice([1, 3, 200, 100_000]))
    k0 = rng.integers(0, min(card, 256), n).astype(np.uint8)
    k1 = rng.integers(-card, card, n).astype(np.int32)
    v = rng.integers(-10**12, 10**12, n)
    w = rng.integers(-(1 << 62), 1 << 62, n)
    k2 = rng.integers(-card, card, n)
    cols = [k0, k1, v, w, k2]
    key_idx = [[0], [1], [0, 1], [1, 0], [], [4], [1, 0, 0]][seed % 7]
    preds = [] if seed % 3 else [(2, "gt", -10**11)]
    gcols = [cu(k0, torch.uint8), cu(k1, torch.int32), cu(v), cu(w), cu(k2)]
    got = T.groupby_agg(gcols, key_idx, AGGS_ALL, preds)
    want = oracle.groupby_agg(cols, key_idx, AGGS_ALL, preds)
    check_groupby(T, got, want, AGGS_ALL)


@pytest.mark.parametrize("e", [0, 22, 23, 24, 25, 46, 47, 48, 49, 60, 62])
@pytest.mark.parametrize("card", [1, 3, 6, 40])
def test_groupby_sum_magnitude_tiers(T, e, card):
    """Sums over warps spanning few runs are reduced as 1, 2 or 3 24-bit pieces chosen
    from the values' magnitude bound; values straddle each tier edge, both signs, and
    products of two factors move the bound across tiers."""
    rng = np.random.default_rng(e * 100 + card)
    n = 70_001
    k = rng.integers(0, card, n)
    hi = 1 << e
    v = rng.integers(-hi, hi + 1, n)
    v[rng.random(n) < 0.01] = hi
    v[rng.random(n) < 0.01] = -hi
    small = rng.integers(-3, 4, n)
    aggs = [("sum", [(1, 0, 1)]), ("sum", [(1, 0, -1)]), ("count", [])]
    if e <= 60:                         # |v * (small + 1)| <= 2^62
        aggs.append(("sum", [(1, 0, 1), (2, 1, 1)]))
    cols = [k, v, small]
    got = T.groupby_agg([cu(c) for c in cols], [0], aggs)
    want = oracle.groupby_agg(cols, [0], aggs)
    check_groupby(T, got, want, aggs)




@pytest.mark.parametrize("card,wide", [(1, False), (2, False), (5, False), (6, False), (5, True)])
def test_groupby_dense_path(T, card, wide, monkeypatch, dense_kernel):
    """Few distinct packed keys (<= 16, packed width <= 16 bits) take the sort-free dense
    kernel; both it and the general tile path (TQP_GROUPBY_DENSE=0) match the oracle."""
    rng = np.random.default_rng(card)
    n = 200_003
    k0 = (rng.integers(0, card, n) * 7 + 60).astype(np.uint8)
    k1 = rng.integers(-2, 1, n).astype(np.int32)
    if wide:   # packed width > 16 bits: the presence pass declines
        k1 = (k1.astype(np.int64) * 100_000).astype(np.int32)
    v = rng.integers(-10**9, 10**9, n)
    w = rng.integers(0, 100, n)
    cols = [k0, k1, v, w]
    gcols = [cu(k0, torch.uint8), cu(k1, torch.int32), cu(v), cu(w)]
    aggs = [("sum", [(2, 0, 1)]), ("sum", [(2, 0, 1), (3, 100, -1)]), ("count", []), ("min", [(2, 0, 1)]),
            ("max", [(3, 5, 1)]), ("avg", [(2, 0, 1)])]
    preds = [(3, "lt", 90)]
    want = oracle.groupby_agg(cols, [0, 1], aggs, preds)
    ctx = T.context()
    ctx.reset_counters()
    ctx.set_profiling(True)
    got = ctx.groupby_agg(gcols, [0, 1], aggs, preds)
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    check_groupby(T, got, want, aggs)
    d_keys = card * 3
    assert ("tqp_groupby_dense" in st) == (d_keys <= 16 and not wide)
    monkeypatch.setenv("TQP_GROUPBY_DENSE", "0")
    ctx.reset_counters()
    ctx.set_profiling(True)
    got = ctx.groupby_agg(gcols, [0, 1], aggs, preds)
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    check_groupby(T, got, want, aggs)
    assert "tqp_groupby_dense" not in st


@pytest.mark.parametrize("where", ["first_unsampled", "middle", "last_row"])
def test_groupby_dense_sampled_presence_miss(T, where, dense_kernel):
    """The dense path takes key presence from a sample of 16-row groups (n > 2^21 rows here,
    so every 3rd group); keys that occur only in unsampled rows are flagged by the dense
    kernel and the presence pass is redone over every row, so no group is lost."""
    rng = np.random.default_rng(21)
    n = 4_000_003
    k = rng.integers(0, 2, n).astype(np.uint8) * 3 + 65
    row = {"first_unsampled": 19, "middle": 2_000_037, "last_row": n - 1}[where]
    k[row] = 90                                  # a group of one row, outside the sample
    k[row + 16 * 4 if row + 64 < n else 0] = 91  # another key in a different (unsampled) group
    v = rng.integers(-10**6, 10**6, n)
    aggs = [("sum", [(1, 0, 1)]), ("count", []), ("max", [(1, 0, 1)])]
    got = T.groupby_agg([cu(k, torch.uint8), cu(v)], [0], aggs)
    want = oracle.groupby_agg([k, v], [0], aggs)
    check_groupby(T, got, want, aggs)
    assert got["n_groups"] == 4


@pytest.mark.parametrize("seed", range(6))
def test_groupby_dense_path_random(T, seed, dense_kernel):
    """Dense path over three key columns (u8, negative i32, u8), != / range predicates that
    may empty some or all groups, and SUM / MIN / MAX / AVG / COUNT of signed expressions."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.choice([1, 511, 512, 513, 70_001, 400_000]))
    k0 = rng.integers(0, 2, n).astype(np.uint8)
    k1 = (rng.integers(-2, 1, n) * 3).astype(np.int32)
    k2 = (rng.integers(0, 2, n) + 200).astype(np.uint8)
    v = rng.integers(-10**9, 10**9, n)
    w = rng.integers(-100, 100, n)
    cols = [k0, k1, k2, v, w]
    gcols = [cu(k0, torch.uint8), cu(k1, torch.int32), cu(k2, torch.uint8), cu(v), cu(w)]
    aggs = [("sum", [(3, 0, 1), (4, 7, -1)]), ("min", [(3, 5, -1)]), ("max", [(4, 0, 1), (4, 0, 1)]),
            ("avg", [(3, 0, 1)]), ("count", []), ("sum", [(4, 0, 1)])]
    preds = [[], [(4, "ne", 0), (3, "gt", -5 * 10**8)], [(1, "ne", -3)], [(4, "gt", 200)]][seed % 4]
    want = oracle.groupby_agg(cols, [0, 1, 2], aggs, preds)
    jit0 = T.jit_counters()
    ctx = T.context()
    ctx.reset_counters()
    ctx.set_profiling(True)
    got = ctx.groupby_agg(gcols, [0, 1, 2], aggs, preds)
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    check_groupby(T, got, want, aggs)
    assert "tqp_groupby_dense" in st   # 12 possible keys, packed width 1 + 3 + 1 bits
    if dense_kernel == "jit":
        jc = T.jit_counters()
        assert jc["available"] and jc["launches"] > jit0["launches"] and jc["failed"] == 0


def test_groupby_dense_bound_fallback(T, dense_kernel):
    """A product the dense path cannot prove exact re-runs on the general path."""
    rng = np.random.default_rng(3)
    n = 100_000
    k = rng.integers(0, 3, n)
    v = rng.integers(-(1 << 40), 1 << 40, n)
    aggs = [("sum", [(1, 0, 1), (1, 0, 1)]), ("count", [])]    # |v*v| up to 2^80: int64 overflow
    with pytest.raises(T.TqpError) as e:
        T.groupby_agg([cu(k), cu(v)], [0], aggs)
    assert e.value.status == T.TQP_ERR_OVERFLOW
    v2 = rng.integers(-(1 << 30), 1 << 30, n)                   # |v*v| < 2^60 but > 2^dense_bits
    aggs = [("sum", [(1, 0, 1), (1, 0, 1)]), ("count", [])]
    got = T.groupby_agg([cu(k), cu(v2)], [0], aggs)
    want = oracle.groupby_agg([k, v2], [0], aggs)
    check_groupby(T, got, want, aggs)


def test_groupby_key_wider_than_64_bits_rejected(T):
    x = cu(np.arange(10))
    with pytest.raises(T.TqpError) as e:
        T.groupby_agg([x, cu(np.arange(10), torch.uint8)], [0, 1], [("count", [])])
    assert e.value.status == T.TQP_ERR_INVALID_ARGUMENT


def test_groupby_high_cardinality(T):
    _, li = tpch_orders_lineitem(0.01, seed=42, device="cuda")
    cols = [li["l_orderkey"], li["l_quantity"], li["l_extendedprice"]]
    aggs = [("sum", [(1, 0, 1)]), ("count", []), ("max", [(2, 0, 1)]), ("avg", [(2, 0, 1)])]
    got = T.groupby_agg(cols, [0], aggs)
    want = oracle.groupby_agg([npy(c) for c in cols], [0], aggs)
    check_groupby(T, got, want, aggs)


def test_groupby_high_cardinality_sf1(T):
    """High cardinality at SF1 (~1.5M groups over 6M lineitem rows): the tiles do not
    reduce, so the group-by takes the global-sort path (Alg. 2 literally); vs the oracle."""
    _, li = tpch_orders_lineitem(1.0, seed=42, device="cuda")
    cols = [li["l_orderkey"], li["l_quantity"], li["l_extendedprice"], li["l_shipdate"]]
    aggs = [("sum", [(1, 0, 1), (2, 0, 1)]), ("count", []), ("min", [(3, 0, 1)]), ("max", [(2, 0, -1)]),
            ("avg", [(1, 0, 1)])]
    preds = [(3, "ge", 9000)]
    got = T.groupby_agg(cols, [0], aggs, preds)
    want = oracle.groupby_agg([npy(c) for c in cols], [0], aggs, preds)
    check_groupby(T, got, want, aggs)


@pytest.mark.parametrize("ncols", [2, 4])
def test_groupby_sort_path_interleaved_gather(T, ncols):
    """The high-cardinality sort path with 2 / 4 distinct factor columns of mixed dtypes
    over 2M rows (above the 2^20-row threshold): the columns are interleaved per row
    (16- / 32-byte records) before the reduction gathers them; no predicate, so the records
    are indexed by row directly. Against the oracle."""
    rng = np.random.default_rng(77 + ncols)
    n = 2_000_003
    k = rng.integers(0, 700_000, n)
    cols = [k]
    gcols = [cu(k)]
    dts = [torch.int64, torch.int32, torch.uint8, torch.int64]
    for c in range(ncols):
        dt = dts[c]
        hi = {torch.uint8: 255, torch.int32: 1 << 20, torch.int64: 1 << 30}[dt]
        v = rng.integers(0 if dt == torch.uint8 else -hi, hi + 1, n)
        cols.append(v.astype(np.int64))
        gcols.append(cu(v, dt))
    aggs = [("sum", [(1, 0, 1)]), ("count", []), ("max", [(2, 3, -1)]), ("sum", [(1, 0, 1), (2, 1, 1)])]
    if ncols == 4:
        aggs += [("min", [(3, 0, 1)]), ("avg", [(4, 0, 1)])]
    got = T.groupby_agg(gcols, [0], aggs)
    check_groupby(T, got, oracle.groupby_agg(cols, [0], aggs), aggs)


def test_groupby_empty_and_global(T):
    e = cu(np.array([], np.int64))
    got = T.groupby_agg([e], [0], [("sum", [(0, 0, 1)])])
    assert got["n_groups"] == 0
    aggs = [("sum", [(0, 0, 1)]), ("count", []), ("min", [(0, 0, 1)]), ("max", [(0, 0, 1)]), ("avg", [(0, 0, 1)])]
    got = T.groupby_agg([e], [], aggs)
    want = oracle.groupby_agg([np.array([], np.int64)], [], aggs)
    check_groupby(T, got, want, aggs)
    x = cu(np.arange(5000))
    got = T.groupby_agg([x], [], aggs, preds=[(0, "lt", -1)])      # nothing passes
    want = oracle.groupby_agg([np.arange(5000)], [], aggs, preds=[(0, "lt", -1)])
    check_groupby(T, got, want, aggs)


def test_groupby_int128_and_overflow(T):
    v = np.full(100_000, (1 << 62) + 12345, np.int64)
    got = T.groupby_agg([cu(v)], [], [("sum", [(0, 0, 1)]), ("avg", [(0, 0, 1)])])
    want = oracle.groupby_agg([v], [], [("sum", [(0, 0, 1)]), ("avg", [(0, 0, 1)])])
    check_groupby(T, got, want, [("sum", []), ("avg", [])])
    with pytest.raises(T.TqpError) as e:
        T.groupby_agg([cu(v)], [], [("sum", [(0, 0, 1), (0, 0, 1)])])
    assert e.value.status == T.TQP_ERR_OVERFLOW


def test_groupby_q1_sf10_full_size(T):
    """BASELINE configs[2]-sized lineitem (60M rows) Q1, bench launch configuration, vs the oracle."""
    _, li = tpch_orders_lineitem(10.0, seed=42, device="cuda")
    cols = columns(li, Q1_COLS)
    got = T.groupby_agg(cols, Q1_KEYS, Q1_AGGS, Q1_PREDS)
    want = oracle.groupby_agg([npy(c) for c in cols], Q1_KEYS, Q1_AGGS, Q1_PREDS)
    check_groupby(T, got, want, Q1_AGGS)


def test_launch_counter_and_profiling(T):
    ctx = T.context()
    ctx.reset_counters()
    ctx.set_profiling(True)
    T.sort(cu(np.arange(10_000)[::-1].copy()))
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    assert ctx.launch_count() >= 3
    assert "tqp_sort_scatter" in st and st["tqp_sort_scatter"][1] >= 1
    assert all(v[1] >= 1 and v[0] > 0 for v in st.values())   # every launch timed
    # filtered: only the scatter launches are timed; the others still count and carry bytes
    ctx.reset_counters()
    ctx.set_profiling(True, only="tqp_sort_scatter")
    T.sort(cu(np.arange(10_000)[::-1].copy()))
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    assert st["tqp_sort_scatter"][1] >= 1 and st["tqp_sort_scatter"][0] > 0
    assert all(v[1] == 0 and v[0] == 0 for k, v in st.items() if k != "tqp_sort_scatter")
    assert ctx.launch_count() >= 3


def _check_f64(got, want, aggs, f64_idx):
    """fp64 aggregates against the oracle: MIN / MAX / COUNT exact; SUM / AVG within the
    bound of an unordered float sum, |d| <= 2 m u sum|v| (u = 2^-53, m rows in the group)."""
    u = 2.0 ** -53
    for a in f64_idx:
        op = aggs[a][0]
        g = got["results"][a].cpu().numpy()
        w = np.array(want["results"][a], dtype=np.float64)
        if op in ("min", "max"):
            assert np.array_equal(g, w), op
            continue
        m = np.array(want["counts"], dtype=np.float64)
        bound = 2 * m * u * np.array(want["abs_sums"][a])
        if op == "avg":
            bound = bound / np.maximum(m, 1) + 4 * u * np.abs(w)
            nan = np.isnan(w)
            assert np.array_equal(np.isnan(g), nan)
            g, w, bound = g[~nan], w[~nan], bound[~nan]
        assert np.all(np.abs(g - w) <= bound + 1e-300), (op, np.max(np.abs(g - w) - bound))


@pytest.mark.parametrize("ng", [1, 6, 300, 50_000])
def test_groupby_f64_aggregates(T, ng):
    """fp64 value columns (TQP_F64) beside integer aggregates, with a fused filter; shared-
    memory accumulators (few groups) and global ones (50K groups)."""
    rng = np.random.default_rng(ng)
    n = 400_003
    k = rng.integers(0, ng, n).astype(np.int32)
    x = rng.normal(0.0, 1e4, n)
    q = rng.integers(0, 5000, n).astype(np.int64)
    d = rng.integers(0, 11, n).astype(np.uint8)
    cols = [cu(k, torch.int32), torch.tensor(x, device="cuda"), cu(q), cu(d, torch.uint8)]
    aggs = [("sum", [(1, 0, 1)]), ("sum", [(2, 0, 1)]), ("avg", [(1, 0, 1)]), ("min", [(1, 0, 1)]),
            ("max", [(1, 0, 1), (3, 100, -1)]), ("sum", [(1, 0, 1), (3, 100, -1), (2, 1, 1)]), ("count", [])]
    preds = [(2, "lt", 4500), (3, "ne", 7)]
    got = T.groupby_agg(cols, [0], aggs, preds)
    wf = oracle.groupby_agg_f64([k, x, q, d], [0], aggs, preds)
    wi = oracle.groupby_agg([k, q, d], [0], [("sum", [(1, 0, 1)])], [(1, "lt", 4500), (2, "ne", 7)])
    assert got["n_groups"] == len(wf["counts"])
    assert npy(got["keys"][0]).tolist() == [int(v) for v in wf["keys"][0]]
    assert T.int128_to_ints(got["results"][1]) == wi["results"][0]
    assert npy(got["results"][6]).tolist() == wf["counts"]
    _check_f64(got, wf, aggs, [0, 2, 3, 4, 5])


def test_groupby_f64_exact_sums_and_global(T):
    """Values on a 2^-4 grid with small magnitudes: every partial sum is exact, so SUM must
    equal the oracle bit for bit whatever the order; no keys; empty global group."""
    rng = np.random.default_rng(5)
    n = 1_000_001
    x = rng.integers(-4000, 4000, n) / 16.0
    k = rng.integers(0, 3, n).astype(np.uint8)
    cols = [cu(k, torch.uint8), torch.tensor(x, device="cuda")]
    aggs = [("sum", [(1, 0, 1)]), ("sum", [(1, 2, -1)]), ("min", [(1, 0, 1)]), ("max", [(1, 0, 1)])]
    for keys in ([0], []):
        got = T.groupby_agg(cols, keys, aggs)
        want = oracle.groupby_agg_f64([k, x], keys, aggs)
        for a in range(4):
            assert npy(got["results"][a]).tolist() == want["results"][a]
    e = T.groupby_agg(cols, [], aggs + [("avg", [(1, 0, 1)]), ("count", [])], [(0, "gt", 5)])
    r = [npy(t).tolist() for t in e["results"]]
    assert r[0] == [0.0] and r[2] == [float("inf")] and r[3] == [float("-inf")] and np.isnan(r[4][0]) and r[5] == [0]


def test_groupby_f64_rejects_f64_keys_and_predicates(T):
    x = torch.randn(100, dtype=torch.float64, device="cuda")
    k = torch.zeros(100, dtype=torch.int64, device="cuda")
    with pytest.raises(T.TqpError):
        T.groupby_agg([x, k], [0], [("count", [])])
    with pytest.raises(T.TqpError):
        T.groupby_agg([k, x], [0], [("count", [])], [(1, "lt", 0)])
    with pytest.raises(T.TqpError):
        T.filter_compact([x], [(0, "lt", 0)])


def test_groupby_merge_partials(T):
    """tqp_groupby_merge over 3 row slices (the multi-GPU gather + final reduce, one process):
    equals the oracle on the whole table, AVG recomputed from merged SUM / COUNT."""
    from paper_2203_01877_b200.dist import _rewrite_aggs
    _, li = tpch_orders_lineitem(0.01, seed=42, device="cuda")
    cols = columns(li, Q1_COLS)
    aggs = Q1_AGGS + [("min", [(3, 0, 1)]), ("max", [(2, 0, 1)])]
    raggs = _rewrite_aggs(aggs)
    n = cols[0].numel()
    cuts = [0, n // 3, (2 * n) // 3, n]
    parts = [T.groupby_agg([c[a:b] for c in cols], Q1_KEYS, raggs, Q1_PREDS) for a, b in zip(cuts, cuts[1:])]
    keys = [torch.cat([p["keys"][k] for p in parts]) for k in range(len(Q1_KEYS))]
    partials = []
    for a, (op, _) in enumerate(aggs):
        partials.append(None if op == "count" else torch.cat([p["results"][a] for p in parts]))
    counts = torch.cat([p["results"][-1] for p in parts])
    got = T.context().groupby_merge(keys, aggs, partials, counts)
    want = oracle.groupby_agg([npy(c) for c in cols], Q1_KEYS, aggs, Q1_PREDS)
    check_groupby(T, got, want, aggs)


# ------------------------------------------------- data-parallel exchange steps

@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 300_001])
@pytest.mark.parametrize("parts", [1, 2, 3, 8, 256])
@pytest.mark.parametrize("dtype", [torch.int64, torch.int32, torch.uint8])
def test_partition_stable_by_key_range(T, n, parts, dtype):
    """tqp_partition = a stable sort by destination (#splitters <= key): numpy's stable
    argsort of the searchsorted destinations, plus bincount counts; keys equal to a
    splitter go to the higher rank; duplicate splitters leave empty destinations."""
    rng = np.random.default_rng(n + parts)
    hi = {torch.int64: 1 << 40, torch.int32: 1 << 30, torch.uint8: 255}[dtype]
    lo = 0 if dtype == torch.uint8 else -hi
    keys = rng.integers(lo, hi, n)
    spl = np.sort(rng.integers(lo, hi, parts - 1))
    if parts > 3:
        spl[1] = spl[2]                     # a duplicate splitter: destination 2 is empty
        keys[: min(n, 5)] = spl[1]          # keys equal to a splitter
    ko, ro, cnt = T.partition(cu(keys, dtype), cu(spl), row_base=1000)
    dest = np.searchsorted(spl, keys, side="right")
    order = np.argsort(dest, kind="stable")
    assert np.array_equal(npy(ko).astype(np.int64), keys[order])
    assert np.array_equal(npy(ro), order + 1000)
    assert np.array_equal(npy(cnt), np.bincount(dest, minlength=parts))


def test_minmax_and_range_splitters(T):
    """Device [min, max] (empty -> [INT64_MAX, INT64_MIN]) and equal-width splitters:
    key k goes to (k - lo) // width, width = (hi - lo) // parts + 1."""
    rng = np.random.default_rng(3)
    k = rng.integers(-(1 << 50), 1 << 50, 100_003)
    mm = npy(T.minmax(cu(k)))
    assert mm.tolist() == [int(k.min()), int(k.max())]
    assert npy(T.minmax(cu(np.array([], np.int64)))).tolist() == [I64_MAX, I64_MIN]
    for parts in (1, 2, 7, 256):
        spl = npy(T.range_splitters(cu(mm), parts))
        w = (int(k.max()) - int(k.min())) // parts + 1
        assert spl.tolist() == [int(k.min()) + (j + 1) * w for j in range(parts - 1)]
        dest = np.searchsorted(spl, k, side="right")
        assert np.array_equal(dest, (k - int(k.min())) // w)
    spl = npy(T.range_splitters(cu(np.array([I64_MIN, I64_MAX])), 4))   # full domain: no overflow
    assert spl[-1] < I64_MAX and np.all(np.diff(spl) > 0)


@pytest.mark.parametrize("dtype", [torch.int64, torch.int32, torch.uint8, torch.float64])
def test_gather(T, dtype):
    rng = np.random.default_rng(4)
    src = rng.integers(0, 200, 50_001)
    idx = rng.integers(0, src.size, 123_457)
    s = torch.as_tensor(src).to(dtype).cuda()
    out = T.gather(s, cu(idx))
    assert torch.equal(out.cpu(), s.cpu()[torch.as_tensor(idx)])


@pytest.mark.parametrize("case", ["random", "zipf", "coarse"])
def test_smj_expand_payload(T, case):
    """createOutput fused into the expansion: payload gathered by the
    oracle's pairs, over the whole output and ragged windows, with and without indices."""
    rng = np.random.default_rng(9)
    if case == "random":
        left, right = rng.integers(0, 3_000, 40_003), rng.integers(0, 3_000, 30_001)
    elif case == "zipf":
        left = zipf_keys(100_000, 20_000, seed=5).numpy()
        right = uniform_keys(100_000, 20_000, seed=6).numpy()
    else:   # heavy keys: the coarse tile-bucket table
        left = rng.permutation(np.concatenate([np.full(30_000, 1), np.arange(3, 503)]))
        right = rng.permutation(np.concatenate([np.arange(3, 503), np.full(40_000, 1)]))
    lp = [cu(rng.integers(-10**12, 10**12, left.size)), cu(rng.integers(0, 255, left.size), torch.uint8)]
    rp = [cu(rng.integers(-2**31, 2**31 - 1, right.size), torch.int32),
          torch.tensor(rng.normal(size=right.size), device="cuda")]
    plan = T.smj_prepare(cu(left), cu(right))
    wl, wr = oracle.smj_join(left, right)
    assert plan.size == len(wl)
    wins = [(0, plan.size), (0, 0), (plan.size // 3, plan.size // 3 + 2049), (plan.size - 7, plan.size)]
    for b, e in wins:
        louts, routs, idx = plan.expand_payload(b, e, lp, rp, indices=(b == 0))
        for c, o in zip(lp, louts):
            assert torch.equal(o.cpu(), c.cpu()[torch.as_tensor(wl[b:e])])
        for c, o in zip(rp, routs):
            assert torch.equal(o.cpu(), c.cpu()[torch.as_tensor(wr[b:e])])
        if b == 0:
            assert np.array_equal(npy(idx[0]), wl[b:e]) and np.array_equal(npy(idx[1]), wr[b:e])
    plan.release()
    (g,), (h,), _ = T.smj_join_payload(cu(left), cu(right), [lp[0]], [rp[0]])
    assert torch.equal(g.cpu(), lp[0].cpu()[torch.as_tensor(wl)])


@pytest.mark.parametrize("nb,np_,span,presorted", [(0, 100, 10, False), (100, 0, 1000, False), (1, 1, 5, False),
                                                   (5_000, 20_000, 20_000, False), (150_000, 1_500_000, 150_000, True),
                                                   (300_001, 123_457, 2_000_000, True), (300_001, 1_000_003, 400_000, False)])
def test_pkfk_outer_build_q13_shape(T, nb, np_, span, presorted):
    """Outer join preserving the build side (Q13: customer LEFT OUTER JOIN orders): the
    oracle's inner pairs in probe order, then every build row without a match, ascending,
    with right = -1. TPC-H-like case: 150K customers, 1.5M orders over 2/3 of them."""
    rng = np.random.default_rng(nb + np_)
    build = rng.permutation(span)[:nb].astype(np.int64)
    if presorted:
        build = np.sort(build)
    if span == 150_000:   # orders reference customers whose key is not 0 mod 3 (TPC-H rule)
        probe = rng.integers(0, span // 3, np_) * 3 + rng.integers(1, 3, np_)
    else:
        probe = rng.integers(-5, span + 5, np_).astype(np.int64)
    lo, ro = T.pkfk_outer_build(cu(build), cu(probe))
    olo, oro = oracle.pkfk_join(build, probe)
    unmatched = np.setdiff1d(np.arange(nb), olo)
    assert np.array_equal(npy(lo), np.concatenate([olo, unmatched]))
    assert np.array_equal(npy(ro), np.concatenate([oro, np.full(len(unmatched), -1)]))


def test_pkfk_outer_build_duplicate_key(T):
    with pytest.raises(T.TqpError) as e:
        T.pkfk_outer_build(cu(np.array([4, 4, 1])), cu(np.array([4, 1])))
    assert e.value.status == T.TQP_ERR_DUPLICATE_BUILD_KEY


@pytest.mark.parametrize("frac", [0.0005, 0.02, 0.5])
def test_smj_sparse_matches_empty_buckets(T, frac):
    """Most left rows without a partner: the expansion's buckets (one per sorted left row)
    are mostly empty, spans of thousands of empty buckets per output tile; checked against
    the oracle over the whole output and windows."""
    rng = np.random.default_rng(int(frac * 1e4))
    n = 400_003
    left = rng.integers(0, 1 << 40, n)
    right = rng.integers(0, 1 << 40, n)
    pick = rng.random(n) < frac
    right[pick] = left[rng.integers(0, n, int(pick.sum()))]
    lo, ro = T.smj_join(cu(left), cu(right))
    olo, oro = oracle.smj_join(left, right)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


@pytest.mark.parametrize("case", ["one_swap", "shuffled_middle", "out_of_range", "sorted", "sorted_i32"])
def test_pkfk_speculative_rank_route(T, case):
    """The build side is taken as sorted from its first and last key alone (the speculative
    rank-bitmap route); a build side that is not in key order after all -- one adjacent swap,
    a shuffled middle, a key outside [first, last] -- must be detected and redone, in join,
    semi and outer mode. Checked against the oracle."""
    rng = np.random.default_rng(len(case))
    nb = 300_017
    build = np.sort(rng.choice(4 * nb, nb, replace=False)).astype(np.int64) + 1000
    if case == "one_swap":
        j = nb // 2
        build[j], build[j + 1] = build[j + 1], build[j]
    elif case == "shuffled_middle":
        mid = build[1:-1].copy()
        rng.shuffle(mid)
        build[1:-1] = mid
    elif case == "out_of_range":
        build[nb // 3] = build[-1] + 5   # above the last key: not sorted, outside [first, last]
        build = np.concatenate([build[: nb // 3], build[nb // 3:]])
    dt = torch.int32 if case == "sorted_i32" else torch.int64
    probe = rng.choice(build, 1_000_003).astype(np.int64)
    probe[::7] = rng.integers(0, 5 * nb, probe[::7].size)   # some misses
    lo, ro = T.pkfk_join(cu(build, dt), cu(probe, dt))
    olo, oro = oracle.pkfk_join(build, probe)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    sel = T.pkfk_semi(cu(build, dt), cu(probe, dt))
    assert np.array_equal(npy(sel), np.unique(oro))
    left = T.pkfk_outer(cu(build, dt), cu(probe, dt))
    want = np.full(probe.size, -1, np.int64)
    want[oro] = olo
    assert np.array_equal(npy(left), want)


@pytest.mark.parametrize("case", ["one_swap", "shuffled_middle", "out_of_range", "sorted"])
def test_poisoned_temporaries(T, case, monkeypatch):
    """Every libtqp temporary filled with garbage when handed out (TQP_ALLOC_POISON=1): a
    kernel reading temporary memory nobody wrote -- e.g. tile counts of probe tiles that
    exited early because the speculative build side was not sorted -- gives wrong results
    or faults here deterministically, not only when the caching allocator happens to hand
    back a used block. The operators' retry and fallback paths against the oracle."""
    monkeypatch.setenv("TQP_ALLOC_POISON", "1")
    ctx = T.Context()
    rng = np.random.default_rng(7 + len(case))
    nb = 200_003
    build = np.sort(rng.choice(4 * nb, nb, replace=False)).astype(np.int64) + 17
    if case == "one_swap":
        build[nb // 2], build[nb // 2 + 1] = build[nb // 2 + 1], build[nb // 2]
    elif case == "shuffled_middle":
        mid = build[1:-1].copy()
        rng.shuffle(mid)
        build[1:-1] = mid
    elif case == "out_of_range":
        build[nb // 3] = build[-1] + 5
    probe = rng.choice(build, 700_001).astype(np.int64)
    probe[::5] = rng.integers(0, 5 * nb, probe[::5].size)
    olo, oro = oracle.pkfk_join(build, probe)
    lo, ro = ctx.pkfk_join(cu(build), cu(probe))
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    lo, ro = ctx.pkfk_join(cu(build), cu(probe), index_dtype=torch.int32)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    sel = ctx.pkfk_semi(cu(build), cu(probe))
    assert np.array_equal(npy(sel), np.unique(oro))
    anti = ctx.pkfk_semi(cu(build), cu(probe), anti=True)
    assert np.array_equal(npy(anti), np.setdiff1d(np.arange(probe.size), oro))
    left = ctx.pkfk_outer(cu(build), cu(probe))
    want = np.full(probe.size, -1, np.int64)
    want[oro] = olo
    assert np.array_equal(npy(left), want)
    bo, po, idx = ctx.pkfk_join_payload(cu(build), cu(probe), build_payload=(cu(build * 3),),
                                        probe_payload=(cu(probe + 1),))
    assert np.array_equal(npy(idx[0]), olo) and np.array_equal(npy(idx[1]), oro)
    assert np.array_equal(npy(bo[0]), build[olo] * 3) and np.array_equal(npy(po[0]), probe[oro] + 1)
    # the other operators' temporaries under the same poisoning
    slo, sro = ctx.smj_join(cu(build), cu(probe))
    xlo, xro = oracle.smj_join(build, probe)
    assert np.array_equal(npy(slo), xlo) and np.array_equal(npy(sro), xro)
    k = (probe % 5).astype(np.uint8)
    aggs = [("sum", [(1, 0, 1)]), ("count", []), ("min", [(1, 0, 1)]), ("max", [(1, 3, -1)])]
    got = ctx.groupby_agg([cu(k, torch.uint8), cu(probe)], [0], aggs, [(1, "gt", 1000)])
    check_groupby(T, got, oracle.groupby_agg([k, probe], [0], aggs, [(1, "gt", 1000)]), aggs)
    got = ctx.groupby_agg([cu(probe), cu(k, torch.uint8)], [0], [("count", []), ("sum", [(1, 0, 1)])])
    check_groupby(T, got, oracle.groupby_agg([probe, k], [0], [("count", []), ("sum", [(1, 0, 1)])]),
                  [("count", []), ("sum", [(1, 0, 1)])])
    mask, sel = ctx.filter_compact([cu(probe)], [(0, "lt", 3 * nb)])
    assert np.array_equal(npy(sel), np.flatnonzero(probe < 3 * nb))
    s = ctx.sort(cu(probe))
    assert np.array_equal(npy(s[0]), np.sort(probe, kind="stable"))


@pytest.mark.parametrize("seed", range(24))
def test_groupby_dense_compiled_plan_fuzz(T, seed, monkeypatch):
    """Random aggregation plans through the plan-compiled dense kernel (jit.cu), each one a
    different generated source: 1-3 key columns of mixed dtypes (u8 / i32 / i64, negative
    values), 1-4 distinct keys (register compares) or 5-16 (id table), 0-4 predicates of
    every comparison kind (folded into interval and != terms, possibly unsatisfiable),
    1-8 (op, expression) pairs with 0-3 factors of mixed dtypes, signs and constants, pairs
    that extend the previous pair's factor list, row counts around the tile edges. Each
    result against the oracle."""
    monkeypatch.setenv("TQP_JIT_MIN_ROWS", "0")
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.choice([1, 511, 512, 513, 2048, 9_999, 65_537, 300_001]))
    n_keys = int(rng.integers(1, 4))
    d_target = int(rng.choice([1, 2, 3, 4, 5, 9, 16]))
    dts = [torch.uint8, torch.int32, torch.int64]
    cols, gcols, kidx = [], [], []
    # key columns: a small domain each, their product near d_target distinct tuples
    per = max(1, round(d_target ** (1.0 / n_keys)))
    width = 0   # the key columns' dtypes fit one 64-bit packed key (the API's limit)
    size = {torch.uint8: 1, torch.int32: 4, torch.int64: 8}
    for k in range(n_keys):
        dt = dts[int(rng.integers(0, 3))]
        if width + size[dt] > 8:
            dt = torch.int32 if width + 4 <= 8 else torch.uint8
        if width + size[dt] > 8:
            break
        width += size[dt]
        lo = 0 if dt == torch.uint8 else int(rng.integers(-50, 50))
        step = int(rng.integers(1, 4))
        v = lo + step * rng.integers(0, per, n)
        cols.append(v.astype(np.int64))
        gcols.append(cu(v, dt))
        kidx.append(len(cols) - 1)
    # value columns
    for _ in range(int(rng.integers(1, 4))):
        dt = dts[int(rng.integers(0, 3))]
        hi = {torch.uint8: 255, torch.int32: 1 << 16, torch.int64: 1 << 18}[dt]   # 3 factors stay < 2^63
        lo = 0 if dt == torch.uint8 else -hi
        v = rng.integers(lo, hi + 1, n)
        cols.append(v.astype(np.int64))
        gcols.append(cu(v, dt))
    vidx = list(range(len(kidx), len(cols)))
    ops = ["lt", "le", "gt", "ge", "eq", "ne"]
    preds = []
    for _ in range(int(rng.integers(0, 5))):
        c = int(rng.integers(0, len(cols)))
        x = int(rng.choice(cols[c])) if n else 0
        preds.append((c, ops[int(rng.integers(0, 6))], x + int(rng.integers(-2, 3))))
    aggs = []
    prev = None
    for _ in range(int(rng.integers(1, 9))):
        op = ["sum", "count", "min", "max", "avg"][int(rng.integers(0, 5))]
        if op == "count":
            aggs.append(("count", []))
            prev = None
            continue
        if prev is not None and len(prev) < 3 and rng.random() < 0.4:   # extends the previous pair's factors
            fs = prev + [(int(rng.choice(vidx)), int(rng.integers(-5, 6)), int(rng.choice([1, -1])))]
        else:
            fs = [(int(rng.choice(vidx)), int(rng.integers(-100, 101)), int(rng.choice([1, -1])))
                  for _ in range(int(rng.integers(0, 3)))]
        aggs.append((op, fs))
        prev = fs if op in ("sum", "avg") else None
    want = oracle.groupby_agg(cols, kidx, aggs, preds)
    jit0 = T.jit_counters()
    ctx = T.context()
    ctx.reset_counters()
    ctx.set_profiling(True)
    got = ctx.groupby_agg(gcols, kidx, aggs, preds)
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    check_groupby(T, got, want, aggs)
    jit1 = T.jit_counters()
    assert jit1["failed"] == jit0["failed"]
    # every dense launch of a plan is the compiled kernel
    assert ("tqp_groupby_dense" in st) == (jit1["launches"] > jit0["launches"])


def test_context_allocator_hooks(T):
    """tqp_ctx_set_allocator (SURVEY §8(b) tqp_alloc_fn / tqp_free_fn): the default Python
    context draws libtqp's temporaries from torch's caching allocator (one HBM pool) and
    trim hands them back; cudaMalloc contexts work the same; an allocator that fails makes
    the operator fail with TQP_ERR_OUT_OF_MEMORY, nothing else; the callbacks come in pairs."""
    import ctypes
    rng = np.random.default_rng(5)
    build = np.sort(rng.choice(10**7, 300_000, replace=False)).astype(np.int64)
    rng.shuffle(build)   # the sort route: plenty of temporaries
    probe = rng.choice(build, 2_000_000)
    olo, oro = oracle.pkfk_join(build, probe)
    b, p = cu(build), cu(probe)
    torch.cuda.synchronize()
    ctx = T.Context(allocator="torch")
    before = torch.cuda.memory_allocated()
    lo, ro = ctx.pkfk_join(b, p)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    if os.environ.get("TQP_ALLOC_EXACT") != "1":   # checked mode frees every temporary at once: no cache
        held = ctx.cached_bytes()
        assert held > 0
        # libtqp's cached blocks are torch allocations (outputs lo / ro come on top)
        assert torch.cuda.memory_allocated() - before >= held
    ctx.trim()
    assert ctx.cached_bytes() == 0
    del lo, ro
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() <= before + 4096
    c2 = T.Context(allocator="cuda")
    lo, ro = c2.pkfk_join(b, p)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
    # an allocator that is always out of memory
    fails = T._ALLOC_T(lambda user, n, dev, s: None)
    frees = T._FREE_T(lambda user, ptr, dev, s: None)
    c3 = T.Context(allocator="cuda")
    assert T._lib.tqp_ctx_set_allocator(c3._h, ctypes.cast(fails, ctypes.c_void_p), None, None) == T.TQP_ERR_INVALID_ARGUMENT
    assert T._lib.tqp_ctx_set_allocator(c3._h, ctypes.cast(fails, ctypes.c_void_p),
                                        ctypes.cast(frees, ctypes.c_void_p), None) == T.TQP_OK
    with pytest.raises(T.TqpError) as e:
        c3.pkfk_join(b, p)
    assert e.value.status == T.TQP_ERR_OUT_OF_MEMORY
    # back to cudaMalloc: the context is still usable
    assert T._lib.tqp_ctx_set_allocator(c3._h, None, None, None) == T.TQP_OK
    lo, ro = c3.pkfk_join(b, p)
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)


@pytest.mark.parametrize("offset", [1, 3])
def test_groupby_dense_unaligned_columns(T, offset, dense_kernel):
    """Columns starting off a 16-byte boundary (views into larger tensors) cannot be staged
    with bulk copies: both dense kernels take the plain cooperative loads for every tile."""
    rng = np.random.default_rng(40 + offset)
    n = 123_457
    k = (rng.integers(0, 3, n + offset) + 65).astype(np.uint8)
    d = rng.integers(-5000, 5000, n + offset).astype(np.int32)
    v = rng.integers(-10**9, 10**9, n + offset)
    cols = [k[offset:], d[offset:], v[offset:]]
    gcols = [cu(k, torch.uint8)[offset:], cu(d, torch.int32)[offset:], cu(v)[offset:]]
    aggs = [("sum", [(2, 0, 1), (1, 7, -1)]), ("count", []), ("min", [(1, 0, 1)]), ("max", [(2, 0, -1)])]
    preds = [(1, "ge", -4000)]
    got = T.groupby_agg(gcols, [0], aggs, preds)
    check_groupby(T, got, oracle.groupby_agg(cols, [0], aggs, preds), aggs)


@pytest.mark.parametrize("case", ["sorted", "one_swap", "shuffled_middle", "high_word", "sorted_dups", "sorted_i32"])
def test_smj_speculative_sorted_left(T, case, monkeypatch):
    """The SMJ takes a left side whose first / last / 2,049 sampled keys are in order as
    sorted without its plan pass; the bucket kernel verifies the order of every adjacent
    pair in the full 64-bit key domain and a left side that is not sorted after all -- one
    adjacent swap, a shuffled middle, a key with another high word that a 32-bit key
    domain would truncate into order -- is prepared again with the sort. Against the
    oracle, with the poisoned allocator (the retry must not read the first attempt's
    temporaries)."""
    monkeypatch.setenv("TQP_ALLOC_POISON", "1")
    ctx = T.Context()
    rng = np.random.default_rng(31 + len(case))
    nl = 150_007
    left = np.sort(rng.choice(4 * nl, nl, replace=not case.endswith("dups"))).astype(np.int64) + 10
    if case == "one_swap":
        j = nl // 2
        left[j], left[j + 1] = left[j + 1], left[j]
    elif case == "shuffled_middle":
        mid = left[1:-1].copy()
        rng.shuffle(mid)
        left[1:-1] = mid
    elif case == "high_word":   # sample-invisible: (1 << 40) + key looks in order when truncated to 32 bits
        j = nl // 2 + 3
        left[j] = (1 << 40) + (left[j - 1] + left[j + 1]) // 2 if left[j + 1] - left[j - 1] > 1 else left[j] + (1 << 40)
    dt = torch.int32 if case == "sorted_i32" else torch.int64
    right = rng.choice(left, 600_001).astype(np.int64)
    right[::9] = rng.integers(0, 5 * nl, right[::9].size)
    if dt == torch.int32:
        left, right = left.astype(np.int32), right.astype(np.int32)
    lo, ro = ctx.smj_join(cu(left, dt), cu(right, dt))
    olo, oro = oracle.smj_join(left.astype(np.int64), right.astype(np.int64))
    assert np.array_equal(npy(lo), olo) and np.array_equal(npy(ro), oro)
