"""The paper's own method on B200: TQP's tensor programs as PyTorch op compositions
(SURVEY.md §8(d) "Paper-method-on-B200 row"). A comparison arm, not the product path:
it times what the paper's algorithms cost on the same GPU and the same SF10 inputs as
bench.py's step, so the gain of the fused libtqp kernels over the paper's own design
is measured on identical hardware.

  PK-FK join   PAPER.md:55-100   both sides sorted descending, build side padded to a
                                 power of two, log2(n') rounds of whole-tensor
                                 index_select binary search, match mask, masked_select
  SMJ          PAPER.md:286-338  Alg. 1: sort both sides, bincount over the key domain,
                                 mul, cumsums, arange(outSize), bucketize(right=True),
                                 div/remainder by rightHist (readings R2-R5)
  Q1 group-by  PAPER.md:340-367  filter (Listing 1 mask) -> Alg. 2: keys concatenated,
                                 stable sort, permute, unique_consecutive(inverse,
                                 counts), segmented sums by scatter_add (int64; decimals
                                 as fixed point, reading R16)
  Q6           PAPER.md:825-851  Listing 1 masks AND-ed, Listing 2 nonzero selection
                                 vector, sum(price * disc) over it

Usage: python tools/paper_torch.py [--steps K] [--warmup W] [--check]  (one GPU)
"""

import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from datagen import tpch_orders_lineitem                                   # noqa: E402
from datagen.queries import Q1_COLS, Q1_PREDS, Q6_COLS, Q6_PREDS, columns  # noqa: E402

_CMP = {"lt": torch.lt, "le": torch.le, "gt": torch.gt, "ge": torch.ge, "eq": torch.eq, "ne": torch.ne}


def pkfk_join(left, right):
    """PK-FK macro with reading R8 (pad below every key)."""
    left_s, left_idx = torch.sort(left, descending=True, stable=True)
    right_s, right_idx = torch.sort(right, descending=True, stable=True)
    n = left_s.shape[0]
    n_prime = 1 << max(1, math.ceil(math.log2(n + 1)))
    min_val = torch.minimum(left_s[-1], right_s[-1])
    padded = torch.cat([left_s, (min_val - 1).expand(n_prime - n)])
    offset = n_prime // 2
    bins = right_s <= padded[offset]
    pos = bins.long() * offset
    offset = (offset + 1) // 2
    for _ in range(int(math.log2(n_prime))):
        bins = right_s <= torch.index_select(padded, 0, pos + offset)
        pos = pos + bins.long() * offset
        offset = offset // 2
    pos = torch.clamp(pos, max=n - 1)
    mask = right_s == torch.index_select(left_s, 0, pos)
    pos = torch.masked_select(pos, mask)
    return torch.index_select(left_idx, 0, pos), torch.masked_select(right_idx, mask)


def smj_join(left, right):
    """Alg. 1, readings R2 (ascending), R3 (right=True), R4 (rem by R)."""
    left_s, left_idx = torch.sort(left, stable=True)
    right_s, right_idx = torch.sort(right, stable=True)
    K = int(torch.maximum(left_s[-1], right_s[-1]).item()) + 1
    lh = torch.bincount(left_s, minlength=K)
    rh = torch.bincount(right_s, minlength=K)
    hm = lh * rh
    cl, cr, cm = torch.cumsum(lh, 0), torch.cumsum(rh, 0), torch.cumsum(hm, 0)
    out_size = int(cm[-1].item())
    offset = torch.arange(out_size, device=left.device)
    b = torch.bucketize(offset, cm, right=True)
    offset = offset - (cm[b] - hm[b])
    R = rh[b]
    div = torch.div(offset, R, rounding_mode="floor")
    rem = offset - div * R
    return left_idx[cl[b] - lh[b] + div], right_idx[cr[b] - rh[b] + rem]


def filter_mask(cols, preds):
    """Listing 1: one comparison mask per predicate, AND-ed."""
    mask = None
    for c, op, v in preds:
        m = _CMP[op](cols[c], v)
        mask = m if mask is None else torch.logical_and(mask, m)
    return mask


def q1_groupby(cols):
    """Q1 as the paper runs it: filter, then Alg. 2 over (returnflag, linestatus)."""
    rf, ls, qty, price, disc, tax, ship = cols
    idx = torch.nonzero(filter_mask(cols, Q1_PREDS)).flatten()                  # Listing 2
    rf, ls, qty, price, disc, tax = (torch.index_select(c, 0, idx) for c in (rf, ls, qty, price, disc, tax))
    grps = torch.stack([rf.long(), ls.long()], dim=1)                            # cat(grpByCols)
    key = grps[:, 0] * 256 + grps[:, 1]                                          # lexicographic
    _, perm = torch.sort(key, stable=True)
    grps = grps[perm]
    qty, price, disc, tax = qty[perm], price[perm], disc[perm], tax[perm]
    uniq, inv, cnt = torch.unique_consecutive(grps, dim=0, return_inverse=True, return_counts=True)
    G = uniq.shape[0]
    disc_price = price * (100 - disc)
    charge = disc_price * (100 + tax)
    sums = []
    for v in (qty, price, disc, disc_price, charge):
        sums.append(torch.zeros(G, dtype=torch.int64, device=v.device).scatter_add_(0, inv, v))
    avgs = [s.double() / cnt.double() for s in (sums[0], sums[1], sums[2])]
    return uniq, sums, avgs, cnt


def q6(cols):
    mask = filter_mask(cols, Q6_PREDS)
    idx = torch.nonzero(mask).flatten()                                          # Listing 2 SV
    price, disc = cols[Q6_COLS.index("l_extendedprice")], cols[Q6_COLS.index("l_discount")]
    return mask, idx, (torch.index_select(price, 0, idx) * torch.index_select(disc, 0, idx)).sum()


def step(ok, lk, q1c, q6c, ev):
    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.append((name, e))
    mark("start")
    r = {"pkfk": pkfk_join(ok, lk)}
    mark("pkfk_join")
    r["smj"] = smj_join(ok, lk)
    mark("smj_join")
    r["q1"] = q1_groupby(q1c)
    mark("q1_groupby")
    m = filter_mask(q6c, Q6_PREDS)
    r["q6_filter"] = (m, torch.nonzero(m).flatten())
    mark("q6_filter")
    r["q6"] = q6(q6c)
    mark("q6_sum")
    return r


def run(steps=5, warmup=2, check=False, sf=10.0):
    dev = torch.device("cuda", 0)
    orders, li = tpch_orders_lineitem(sf, seed=42, device=dev)
    ok, lk = orders["o_orderkey"], li["l_orderkey"]
    q1c, q6c = columns(li, Q1_COLS), columns(li, Q6_COLS)
    for _ in range(warmup):
        step(ok, lk, q1c, q6c, [])
    torch.cuda.synchronize()
    ev, op_ms = [], {}
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        res = step(ok, lk, q1c, q6c, ev)
    t1.record()
    torch.cuda.synchronize()
    for i in range(1, len(ev)):
        if ev[i][0] != "start":
            op_ms[ev[i][0]] = op_ms.get(ev[i][0], 0.0) + ev[i - 1][1].elapsed_time(ev[i][1]) / steps
    ms = t0.elapsed_time(t1) / steps
    out = {"impl": "paper-torch", "metric": "lineitem rows per second through the hot-path step",
           "value": lk.numel() / (ms * 1e-3), "unit": "rows/s", "ms_per_step": ms,
           "op_ms": {k: round(v, 3) for k, v in op_ms.items()}, "steps": steps, "warmup": warmup,
           "config": {"workload": f"tpch_sf{sf:g}_hot_path (same step as bench.py, paper's tensor programs "
                                  "as torch ops on the same GPU)"}}
    if check:   # sanity: same results as libtqp (not a parity pin: both are checked against the oracle elsewhere)
        import paper_2203_01877_b200 as T
        lo, ro = T.pkfk_join(ok, lk)
        plo, pro = res["pkfk"]
        o1, o2 = torch.argsort(ro), torch.argsort(pro)
        same_pkfk = torch.equal(lo[o1], plo[o2]) and torch.equal(ro[o1], pro[o2])
        sl, sr = T.smj_join(ok, lk)
        same_smj = torch.equal(sl, res["smj"][0]) and torch.equal(sr, res["smj"][1])
        mask, sel = T.filter_compact(q6c, Q6_PREDS)
        same_q6 = torch.equal(sel, res["q6_filter"][1]) and torch.equal(mask.bool(), res["q6_filter"][0])
        out["check"] = {"pkfk_pairs_equal_as_sets": bool(same_pkfk), "smj_equal": bool(same_smj),
                        "q6_filter_equal": bool(same_q6)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    print(json.dumps(run(a.steps, a.warmup, a.check, a.sf)))


if __name__ == "__main__":
    main()
