"""Per-operator timing on SF10 (dev tool): each operator alone, repeated, with the
library's per-kernel CUDA-event stats and host wall time, to separate kernel time
from host-side gaps (syncs, allocations)."""

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_01877_b200 as T                                   # noqa: E402
from datagen import tpch_orders_lineitem                            # noqa: E402
from datagen.queries import (Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS,   # noqa: E402
                             Q6_AGGS, Q6_COLS, Q6_PREDS, columns)


def main():
    sf = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
    reps = 5
    orders, li = tpch_orders_lineitem(sf, seed=42, device="cuda")
    ok, lk = orders["o_orderkey"], li["l_orderkey"]
    q1, q6 = columns(li, Q1_COLS), columns(li, Q6_COLS)
    lk32 = lk.to(torch.int32)
    ctx = T.context()
    g = torch.Generator(device="cuda").manual_seed(7)
    ok_shuf = ok[torch.randperm(ok.numel(), device="cuda", generator=g)]   # general route (slot table)
    ok_half = ok[::2].contiguous()                                           # ~50 % of probe rows match
    ops = {
        "pkfk_join_shuffled_build": lambda: ctx.pkfk_join(ok_shuf, lk),
        "pkfk_join_half_match": lambda: ctx.pkfk_join(ok_half, lk),
        "sort_build": lambda: ctx.sort(ok),
        "sort_probe": lambda: ctx.sort(lk),
        "cub_sort_probe_i64": lambda: torch.sort(lk, stable=True),
        "cub_sort_probe_i32": lambda: torch.sort(lk32, stable=True),
        "pkfk_join": lambda: ctx.pkfk_join(ok, lk),
        "pkfk_join_i32": lambda: ctx.pkfk_join(ok, lk, index_dtype=torch.int32),
        "pkfk_small_build": lambda: ctx.pkfk_join(ok[:65536], lk),
        "pkfk_hash_ablation": lambda: ctx.pkfk_join_hash(ok, lk),
        "smj_join": lambda: ctx.smj_join(ok, lk),
        "q1_groupby": lambda: ctx.groupby_agg(q1, Q1_KEYS, Q1_AGGS, Q1_PREDS),
        "q6_filter": lambda: ctx.filter_compact(q6, Q6_PREDS),
        "q6_sum": lambda: ctx.groupby_agg(q6, [], Q6_AGGS, Q6_PREDS),
        # high cardinality (general sorted-tile path): 15M groups
        "gb_orderkey": lambda: ctx.groupby_agg([lk, li["l_quantity"], li["l_extendedprice"]], [0],
                                               [("sum", [(1, 0, 1)]), ("count", []), ("max", [(2, 0, 1)])]),
    }
    out = {}
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    for name, f in ops.items():
        if only and name not in only:
            continue
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        ctx.reset_counters()
        ctx.set_profiling(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps * 1e3
        st = ctx.kernel_stats()
        ctx.set_profiling(False)
        out[name] = {"event_ms": e0.elapsed_time(e1) / reps, "wall_ms": wall,
                     "kernel_ms": sum(v[0] for v in st.values()) / reps,
                     "kernels": {k: [round(v[0] / reps, 4), v[1] / reps, round(v[2] / max(v[0], 1e-9) / 1e6, 1)]
                                 for k, v in sorted(st.items(), key=lambda kv: -kv[1][0])}}
        print(name, json.dumps(out[name]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
