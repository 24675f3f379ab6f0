"""CPU oracle for the TQP hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around oracle/oracle.c (plain single-threaded C; see its
header for the definition each function writes out and the PAPER.md passage it
follows). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package. It imports nothing from the
product package `paper_2203_01877_b200` and shares no code with it.

All column inputs are widened to int64 numpy arrays here (u8 as unsigned
values, i32/i64 signed), which preserves every comparison and every value.
"""

import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "oracle.c")
_LIB = os.path.join(_DIR, "liboracle.so")

OK, ERR_ARG, ERR_DUP, ERR_OOM, ERR_OVERFLOW, ERR_CAPACITY = 0, 1, 2, 3, 5, 6
LT, LE, GT, GE, EQ, NE = range(6)
SUM, COUNT, MIN, MAX, AVG = range(5)
_OPS = {"lt": LT, "le": LE, "gt": GT, "ge": GE, "eq": EQ, "ne": NE,
        "<": LT, "<=": LE, ">": GT, ">=": GE, "==": EQ, "!=": NE}
_AGGS = {"sum": SUM, "count": COUNT, "min": MIN, "max": MAX, "avg": AVG}


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"oracle {what}: status {status}")
        self.status = status


def build(force=False):
    """Compile liboracle.so with gcc (plain -O2, no vectorisation flags needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Pred(ctypes.Structure):
    _fields_ = [("col", ctypes.c_int32), ("op", ctypes.c_int32), ("value", ctypes.c_int64)]


class _Agg(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("n_factors", ctypes.c_int32), ("col", ctypes.c_int32 * 3),
                ("sign", ctypes.c_int32 * 3), ("add", ctypes.c_int64 * 3)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
    return _lib


def _i64(a):
    a = np.asarray(a)
    if a.dtype == np.uint8 or a.dtype == np.bool_:
        a = a.astype(np.int64)
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(st, what, allow=()):
    if st != OK and st not in allow:
        raise OracleError(st, what)
    return st


# ---------------------------------------------------------------- operators

def sort(keys, descending=False):
    """Stable (key, row) order -> (sorted_keys, perm). PAPER.md:296-297, :352."""
    k = _i64(keys)
    n = k.size
    perm = np.empty(n, np.int64)
    srt = np.empty(n, np.int64)
    _check(_L().oracle_sort(_p(k), ctypes.c_int64(n), ctypes.c_int(int(bool(descending))), _p(perm), _p(srt)), "sort")
    return srt, perm


def pkfk_join(build_keys, probe_keys):
    """{(b, p): build[b] == probe[p]} in probe-row order. PAPER.md:55-100."""
    b, p = _i64(build_keys), _i64(probe_keys)
    lo = np.empty(max(p.size, 1), np.int64)
    ro = np.empty(max(p.size, 1), np.int64)
    m = ctypes.c_int64(0)
    _check(_L().oracle_pkfk_join(_p(b), ctypes.c_int64(b.size), _p(p), ctypes.c_int64(p.size),
                                 _p(lo), _p(ro), ctypes.byref(m)), "pkfk_join")
    return lo[:m.value].copy(), ro[:m.value].copy()


def nested_join(left, right):
    """Brute-force O(n*m) pairs in (l, r) loop order."""
    l, r = _i64(left), _i64(right)
    m = ctypes.c_int64(0)
    st = _L().oracle_nested_join(_p(l), ctypes.c_int64(l.size), _p(r), ctypes.c_int64(r.size),
                                 None, None, ctypes.c_int64(0), ctypes.byref(m))
    _check(st, "nested_join", allow=(ERR_CAPACITY,))
    lo = np.empty(max(m.value, 1), np.int64)
    ro = np.empty(max(m.value, 1), np.int64)
    _check(_L().oracle_nested_join(_p(l), ctypes.c_int64(l.size), _p(r), ctypes.c_int64(r.size),
                                   _p(lo), _p(ro), ctypes.c_int64(m.value), ctypes.byref(m)), "nested_join")
    return lo[:m.value].copy(), ro[:m.value].copy()


def smj_count(left, right):
    """Exact output size sum_k L_k * R_k (Alg.1 l.5-9)."""
    l, r = _i64(left), _i64(right)
    m = ctypes.c_int64(0)
    _check(_L().oracle_smj_count(_p(l), ctypes.c_int64(l.size), _p(r), ctypes.c_int64(r.size), ctypes.byref(m)),
           "smj_count")
    return m.value


def smj_join(left, right):
    """All (l, r) with left[l] == right[r] in (key, l, r) order."""
    l, r = _i64(left), _i64(right)
    size = smj_count(l, r)
    lo = np.empty(max(size, 1), np.int64)
    ro = np.empty(max(size, 1), np.int64)
    m = ctypes.c_int64(0)
    _check(_L().oracle_smj_join(_p(l), ctypes.c_int64(l.size), _p(r), ctypes.c_int64(r.size),
                                _p(lo), _p(ro), ctypes.c_int64(size), ctypes.byref(m)), "smj_join")
    return lo[:m.value].copy(), ro[:m.value].copy()


def smj_window(left, right, begin, end):
    """Pairs at output offsets [begin, end) by the per-offset route."""
    l, r = _i64(left), _i64(right)
    k = max(end - begin, 1)
    lo = np.empty(k, np.int64)
    ro = np.empty(k, np.int64)
    _check(_L().oracle_smj_window(_p(l), ctypes.c_int64(l.size), _p(r), ctypes.c_int64(r.size),
                                  ctypes.c_int64(begin), ctypes.c_int64(end), _p(lo), _p(ro)), "smj_window")
    return lo[:end - begin].copy(), ro[:end - begin].copy()


def mix64(x):
    """splitmix64's finaliser on uint64 (the mix of the fused expansion consumer,
    include/tqp.h tqp_smj_expand_checksum; a definition of ours, not the paper's).
    Pinned by splitmix64's published outputs (tests/test_oracle_joins.py)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def smj_checksum(left, right, begin, end):
    """The fused consumer over output offsets [begin, end): the pairs of smj_window
    (PAPER.md:310-330), then (sum_j mix64(mix64((l_j << 32) | r_j) ^ j), sum_j l_j,
    sum_j r_j), each mod 2^64."""
    lo, ro = smj_window(left, right, begin, end)
    lu, ru = lo.astype(np.uint64), ro.astype(np.uint64)
    j = np.arange(begin, end, dtype=np.uint64)
    h = mix64(mix64((lu << np.uint64(32)) | ru) ^ j)
    return (int(h.sum(dtype=np.uint64)), int(lu.sum(dtype=np.uint64)), int(ru.sum(dtype=np.uint64)))


def _preds(preds):
    arr = (_Pred * max(len(preds), 1))()
    for i, (c, op, v) in enumerate(preds):
        arr[i].col = c
        arr[i].op = _OPS[op] if isinstance(op, str) else int(op)
        arr[i].value = int(v)
    return arr


def _cols(cols):
    cs = [_i64(c) for c in cols]
    ptrs = (ctypes.c_void_p * max(len(cs), 1))(*[c.ctypes.data for c in cs])
    return cs, ptrs


def filter_compact(cols, preds):
    """Listing 1 mask and Listing 2 selection vector.
    preds: list of (col, op, value). Returns (mask u8, sel int64)."""
    cs, ptrs = _cols(cols)
    n = cs[0].size if cs else 0
    mask = np.empty(max(n, 1), np.uint8)
    sel = np.empty(max(n, 1), np.int64)
    m = ctypes.c_int64(0)
    pa = _preds(preds)
    _check(_L().oracle_filter(ptrs, ctypes.c_int(len(cs)), ctypes.c_int64(n), pa, ctypes.c_int(len(preds)),
                              _p(mask), _p(sel), ctypes.byref(m)), "filter")
    return mask[:n].copy(), sel[:m.value].copy()


def groupby_agg(cols, key_idx, aggs, preds=()):
    """Sort-based group-by reference (Alg. 2), plain definition.

    aggs: list of (op, [(col, add, sign), ...]) -- value = prod(add + sign*col).
    Returns dict(keys=[np arrays per key col], results=[per agg: python ints
    (SUM as exact int), ints (COUNT/MIN/MAX) or floats (AVG)], n_groups=G)."""
    cs, ptrs = _cols(cols)
    n = cs[0].size if cs else 0
    ki = (ctypes.c_int * max(len(key_idx), 1))(*key_idx)
    aa = (_Agg * max(len(aggs), 1))()
    for i, (op, factors) in enumerate(aggs):
        aa[i].op = _AGGS[op] if isinstance(op, str) else int(op)
        aa[i].n_factors = len(factors)
        for f, (c, add, sign) in enumerate(factors):
            aa[i].col[f] = c
            aa[i].add[f] = add
            aa[i].sign[f] = sign
    pa = _preds(list(preds))
    G = ctypes.c_int64(0)
    st = _L().oracle_groupby(ptrs, ctypes.c_int(len(cs)), ctypes.c_int64(n), ki, ctypes.c_int(len(key_idx)),
                             pa, ctypes.c_int(len(preds)), aa, ctypes.c_int(len(aggs)),
                             ctypes.c_int64(0), ctypes.byref(G), None, None)
    _check(st, "groupby", allow=(ERR_CAPACITY,))
    g = G.value
    keys = np.empty(max(g * len(key_idx), 1), np.int64)
    res = np.empty(max(g * len(aggs) * 2, 1), np.int64)
    _check(_L().oracle_groupby(ptrs, ctypes.c_int(len(cs)), ctypes.c_int64(n), ki, ctypes.c_int(len(key_idx)),
                               pa, ctypes.c_int(len(preds)), aa, ctypes.c_int(len(aggs)),
                               ctypes.c_int64(g), ctypes.byref(G), _p(keys), _p(res)), "groupby")
    keys = keys[:g * len(key_idx)].reshape(g, len(key_idx))
    res = res[:g * len(aggs) * 2].reshape(g, len(aggs), 2)
    out = []
    for a, (op, _) in enumerate(aggs):
        o = _AGGS[op] if isinstance(op, str) else int(op)
        if o == SUM:
            out.append([int(np.uint64(res[i, a, 0])) + (int(res[i, a, 1]) << 64) for i in range(g)])
        elif o == AVG:
            out.append([float(res[i, a, 0:1].view(np.float64)[0]) for i in range(g)])
        else:
            out.append([int(res[i, a, 0]) for i in range(g)])
    return {"n_groups": g, "keys": [keys[:, k].copy() for k in range(len(key_idx))], "results": out}


_NP_OPS = {LT: np.less, LE: np.less_equal, GT: np.greater, GE: np.greater_equal, EQ: np.equal, NE: np.not_equal}


def groupby_agg_f64(cols, key_idx, aggs, preds=()):
    """Group-by whose aggregates take float64 factor columns (include/tqp.h TQP_F64;
    SURVEY.md §8(f) NEXT 4), written out in numpy: rows passing the AND of the
    predicates, grouped by the key tuple in ascending order (Alg. 2,
    PAPER.md:340-367), value per row = prod_f (add_f + sign_f * x_f) in float64, left to
    right. SUM = the correctly rounded sum of the group's values (math.fsum), MIN / MAX,
    COUNT = rows, AVG = SUM / COUNT. Returns dict(keys, results, abs_sums) with
    abs_sums[a][g] = sum of |v| (the scale of an unordered float sum's error bound)."""
    import math
    cols = [np.asarray(c) for c in cols]
    n = cols[0].size if cols else 0
    m = np.ones(n, dtype=bool)
    for c, op, v in preds:
        o = _OPS[op] if isinstance(op, str) else int(op)
        m &= _NP_OPS[o](cols[c].astype(np.int64), np.int64(v))
    rows = np.nonzero(m)[0]
    if key_idx:
        kt = np.stack([cols[k].astype(np.int64)[rows] for k in key_idx], axis=1)
        uk, inv = np.unique(kt, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        G = uk.shape[0]
        keys = [uk[:, j] for j in range(len(key_idx))]
    else:
        inv = np.zeros(rows.size, dtype=np.int64)
        G = 1
        keys = []
    members = [rows[inv == g] for g in range(G)] if key_idx else [rows]
    results, abs_sums = [], []
    for op, factors in aggs:
        o = _AGGS[op] if isinstance(op, str) else int(op)
        v = np.ones(n, dtype=np.float64)
        for f, (c, add, sign) in enumerate(factors):
            t = np.float64(add) + np.float64(sign) * cols[c].astype(np.float64)
            v = t if f == 0 else v * t
        out = []
        for mem in members:
            x = v[mem]
            if o == COUNT:
                out.append(int(mem.size))
            elif o == SUM:
                out.append(math.fsum(x.tolist()))
            elif o == AVG:
                out.append(math.fsum(x.tolist()) / mem.size if mem.size else float("nan"))
            elif o == MIN:
                out.append(float(x.min()) if mem.size else float("inf"))
            else:
                out.append(float(x.max()) if mem.size else float("-inf"))
        results.append(out)
        abs_sums.append([math.fsum(np.abs(v[mem]).tolist()) for mem in members])
    return {"keys": keys, "results": results, "abs_sums": abs_sums, "counts": [int(x.size) for x in members]}

