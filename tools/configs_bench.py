"""Per-configuration timings for every BASELINE.json config on one B200:
small configs as latency (launch-bound), large ones as throughput. Not the driver's bench
line (bench.py times the SF10 hot-path step); this is the context table in DESIGN.md §10.

usage: python tools/configs_bench.py [--out profiles/configs_r01.json] [--skip-sf100]
"""

import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_01877_b200 as T                                   # noqa: E402
from datagen import tpch_orders_lineitem, uniform_keys, zipf_keys   # noqa: E402
from datagen.queries import (Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS,   # noqa: E402
                             Q6_AGGS, Q6_COLS, Q6_PREDS, columns)


def timed(f, reps=20, warm=3):
    """Median and min device time (ms) of f() over reps runs, CUDA events, one run each."""
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def tpch_ops(sf, which, reps):
    orders, li = tpch_orders_lineitem(sf, seed=42, device="cuda")
    ok, lk = orders["o_orderkey"], li["l_orderkey"]
    q1, q6 = columns(li, Q1_COLS), columns(li, Q6_COLS)
    ops = {"pkfk_join": lambda: T.pkfk_join(ok, lk),
           "q1_groupby": lambda: T.groupby_agg(q1, Q1_KEYS, Q1_AGGS, Q1_PREDS),
           "q6_filter": lambda: T.filter_compact(q6, Q6_PREDS),
           "q6_sum": lambda: T.groupby_agg(q6, [], Q6_AGGS, Q6_PREDS)}
    out = {"lineitem_rows": lk.numel(), "orders_rows": ok.numel()}
    for name in which:
        med, mn = timed(ops[name], reps)
        out[name] = {"median_ms": round(med, 4), "min_ms": round(mn, 4),
                     "rows_per_s": lk.numel() / (med * 1e-3)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-sf100", action="store_true")
    a = ap.parse_args()
    res = {}
    res["c0_sf0.01"] = tpch_ops(0.01, ["pkfk_join", "q1_groupby"], 50)
    res["c1_sf1"] = tpch_ops(1.0, ["q6_filter", "q6_sum", "q1_groupby"], 30)
    res["c2_sf10"] = tpch_ops(10.0, ["pkfk_join"], 20)
    # c3: Zipf(s=1) left x uniform right, 100M x 100M: prepare + full expand
    n = 100_000_000
    left = zipf_keys(n, n, seed=42, device="cuda")
    right = uniform_keys(n, n, seed=43, device="cuda")
    ctx = T.context()

    def smj():
        plan = ctx.smj_prepare(left, right)
        lo, ro = plan.expand(0, plan.size)
        plan.release()
        return plan.size
    size = smj()
    med, mn = timed(smj, 5, 1)
    res["c3_zipf_smj_100m"] = {"pairs": size, "median_ms": round(med, 3), "min_ms": round(mn, 3),
                               "pairs_per_s": size / (med * 1e-3), "input_rows_per_s": 2 * n / (med * 1e-3)}
    del left, right
    torch.cuda.empty_cache()
    # c3b: config 4 as stated, both sides Zipf(s=1) over [0, 1e8): outSize ~4.6e13 pairs
    # cannot be materialised; prepare timed fully, then 4 windows of 2^30 pairs consumed
    # by the fused checksum (offset 0 + 3 seeded offsets), and one 2^28-pair window
    # materialised for comparison
    left = zipf_keys(n, n, seed=42, device="cuda")
    right = zipf_keys(n, n, seed=43, stream=101, device="cuda")
    holder = {}

    def prep():
        if "p" in holder:
            holder["p"].release()
        holder["p"] = ctx.smj_prepare(left, right)
    prep()
    med_p, min_p = timed(prep, 5, 1)
    plan = holder["p"]
    W = 1 << 30
    g = torch.Generator().manual_seed(4)
    offs = [0] + [int(torch.randint(0, plan.size - W, (1,), generator=g)) for _ in range(3)]
    wins = []
    for b in offs:
        med, mn = timed(lambda: plan.checksum(b, b + W), 3, 1)
        wins.append({"begin": b, "median_ms": round(med, 3), "pairs_per_s": W / (med * 1e-3)})
    buf = (torch.empty(1 << 28, dtype=torch.int64, device="cuda"), torch.empty(1 << 28, dtype=torch.int64, device="cuda"))
    med_m, _ = timed(lambda: plan.expand(offs[1], offs[1] + (1 << 28), out=buf), 3, 1)
    res["c3b_both_zipf_100m"] = {"out_size": plan.size, "prepare_median_ms": round(med_p, 3),
                                 "checksum_windows_2e30": wins,
                                 "materialised_2e28_ms": round(med_m, 3),
                                 "materialised_pairs_per_s": (1 << 28) / (med_m * 1e-3)}
    plan.release()
    del left, right, buf
    torch.cuda.empty_cache()
    if not a.skip_sf100:
        res["c4_sf100_one_gpu"] = tpch_ops(100.0, ["pkfk_join", "q1_groupby"], 5)
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
