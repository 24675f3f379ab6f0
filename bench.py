#!/usr/bin/env python
"""bench.py -- one step = one pass of the whole TQP hot path
over one TPC-H-shaped batch, timed on B200.

Step (per rank, BASELINE.json configs[2] size: SF10 = 15M orders / ~60M lineitem):
  1. tqp_pkfk_join   lineitem.l_orderkey -> orders.o_orderkey      (a1-a4: build radix sort,
                                                                      bracket probe, compaction)
  2. tqp_smj_*       generic m:n sort-merge join of the same keys  (a1-a2, a5-a7)
  3. tqp_groupby_agg TPC-H Q1: filter + group by (returnflag, linestatus), 8 aggregates (a8-a10)
  4. tqp_filter_compact  TPC-H Q6 predicates -> bitmap + selection vector (a10)
  5. tqp_groupby_agg Q6 revenue: fused filter + sum (n_keys = 0)
Multi-GPU (torchrun, one process per GPU): each rank holds an SF10-sized slice of an
SF(10*N) dataset -- its orders rows and a lineitem slice whose orders are spread over every
rank (--placement exchange, the default). The PK-FK join then exchanges
over NCCL (co-partition all_to_all of (key, global row) by key range, or a broadcast build,
whichever the byte model picks), the SMJ runs the distributed sort-merge join (sampled
splitters, heavy keys split by output range), and the Q1/Q6 partial aggregates are
all-gathered and merged by libtqp (tqp_groupby_merge). --placement local keeps each
rank's lineitem with its own orders (no join exchange: the upper bound). scaling = "weak".

value = lineitem rows processed per second by the whole job (all ranks), device-timed with
CUDA events, max over ranks. Inputs (2.8 GB/rank) are larger than L2 (126 MB).
`--impl reference` times the CPU oracle (oracle/, single-threaded C) on a bounded sample.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from datagen import tpch_orders_lineitem                                    # noqa: E402
from datagen.queries import (Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS, Q6_AGGS,  # noqa: E402
                             Q6_COLS, Q6_PREDS, columns)
from datagen.tpch import orders_count                                       # noqa: E402

BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASE["metric"]
SF_PER_RANK = 10.0


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
                for i, n in enumerate(names):
                    if s[2 + i].lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ data

SEED = 42


def make_data(rank, world, device, layout, placement="local"):
    n_o = orders_count(SF_PER_RANK)
    orders, li = tpch_orders_lineitem(SF_PER_RANK * world, seed=SEED, device=device, layout=layout,
                                      order_range=(rank * n_o, (rank + 1) * n_o))
    if placement == "exchange" and world > 1:   # lineitem's orders spread over every rank
        from datagen.tpch import spread_orderkeys
        li["l_orderkey"], _ = spread_orderkeys(li["l_parent"], rank, world)
    return orders, li


def compulsory_bytes(hp, out):
    """SURVEY.md §8(d) compulsory bytes per operator of one step (int64 keys and indices):
    sort(n) = 24 n; PK-FK = sort(n_b) + 8 n_b + 8 n_p + 16 m; SMJ = sort(n_l) + sort(n_r)
    + 8 (n_l + n_r) + 16 outSize; group-by / filter = the bytes of the columns read per row
    (+ the bitmap and selection vector for the filter)."""
    es = lambda cols: sum(c.element_size() for c in {id(c): c for c in cols}.values())   # noqa: E731
    nb, npr, n = hp.ok.numel(), hp.lk.numel(), hp.n
    m = out["pkfk"][0].numel()
    osz = out["smj"][0].numel()
    return {
        "pkfk_join": 24 * nb + 8 * nb + 8 * npr + 16 * m,
        "smj_join": 24 * nb + 24 * npr + 8 * (nb + npr) + 16 * osz,
        "q1_groupby": es(hp.q1) * n,
        "q6_filter": es(hp.q6[:3]) * n + n + 8 * out["q6_sel"].numel(),
        "q6_sum": es(hp.q6) * n,
    }


def q_avg_rewrite(aggs):
    """Distributed AVG: compute SUM (same expression) + one COUNT per rank; merge recomputes AVG."""
    out = []
    for op, f in aggs:
        out.append(("sum", f) if op == "avg" else (op, f))
    out.append(("count", []))
    return out


# ------------------------------------------------------------------ GPU step

class HotPath:
    def __init__(self, T, orders, li, world, placement="local", streams=1, agg_group=None):
        self.T = T
        self.ctx = T.context()
        self.world = world
        self.exchange = placement == "exchange" and world > 1
        self.strategy = None
        self.transport = "nccl"   # co-partition exchange: NCCL all_to_all, or "p2p" (fused partition + peer stores)
        self.pkfk_strategy = "auto"
        # streams = 2: the aggregation queries (Q1, Q6 filter, Q6 sum) run on a second
        # stream from a worker thread with their own libtqp context, concurrently with the
        # joins (inter-operator parallelism: independent operators fill each other's
        # sync gaps and leave-over bandwidth); agg_group: their own process group at N > 1
        self.streams = streams
        self.agg_group, self.join_group = agg_group if agg_group else (None, None)
        if streams > 1:
            import concurrent.futures
            self.s2 = torch.cuda.Stream()
            with torch.cuda.stream(self.s2):
                self.ctx2 = T.Context()
            self.pool = concurrent.futures.ThreadPoolExecutor(max_workers=2)
        if streams > 2:   # the PK-FK join on a third stream, concurrently with the SMJ
            self.s3 = torch.cuda.Stream()
            with torch.cuda.stream(self.s3):
                self.ctx3 = T.Context()
        self.ok = orders["o_orderkey"]
        self.lk = li["l_orderkey"]
        self.q1 = columns(li, Q1_COLS)
        self.q6 = columns(li, Q6_COLS)
        self.n = self.lk.numel()
        self.op_ms = {}
        self._ev = []

    def _mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self._ev.append((name, e))

    def groupby(self, cols, keys, aggs, preds, ctx=None, group=None):
        ctx = ctx or self.ctx
        if self.world == 1:
            return ctx.groupby_agg(cols, keys, aggs, preds)
        from paper_2203_01877_b200 import dist
        return dist.groupby_agg(ctx, cols, keys, aggs, preds, group=group)

    def _aggregations(self, q1, q6):
        """Q1 group-by, Q6 filter (BM + SV), Q6 fused filter + sum on the second stream."""
        with torch.cuda.stream(self.s2):
            r1 = self.groupby(q1, Q1_KEYS, Q1_AGGS, Q1_PREDS, ctx=self.ctx2, group=self.agg_group)
            mask, sel = self.ctx2.filter_compact(q6, Q6_PREDS)
            r6 = self.groupby(q6, [], Q6_AGGS, Q6_PREDS, ctx=self.ctx2, group=self.agg_group)
        return r1, mask, sel, r6

    def _pkfk(self, ok, lk):
        with torch.cuda.stream(self.s3):
            if self.exchange:
                from paper_2203_01877_b200 import dist
                self.strategy, lo, ro = dist.pkfk_join_shuffled(self.ctx3, ok, lk, group=self.join_group,
                                                                strategy=self.pkfk_strategy, transport=self.transport)
            else:
                lo, ro = self.ctx3.pkfk_join(ok, lk)
        return lo, ro

    def step(self, ok=None, lk=None, q1=None, q6=None):
        ok = self.ok if ok is None else ok
        lk = self.lk if lk is None else lk
        q1 = self.q1 if q1 is None else q1
        q6 = self.q6 if q6 is None else q6
        c = self.ctx
        if self.streams > 1:   # concurrent: joins here, aggregations on the second stream
            main = torch.cuda.current_stream()
            self.s2.wait_stream(main)
            fut = self.pool.submit(self._aggregations, q1, q6)
            if self.streams > 2:
                self.s3.wait_stream(main)
                fut3 = self.pool.submit(self._pkfk, ok, lk)
            if self.exchange:
                from paper_2203_01877_b200 import dist
                if self.streams == 2:
                    self.strategy, lo, ro = dist.pkfk_join_shuffled(c, ok, lk, strategy=self.pkfk_strategy, transport=self.transport)
                sl, sr = dist.smj_join_copartition(c, ok, lk)
            else:
                if self.streams == 2:
                    lo, ro = c.pkfk_join(ok, lk)
                plan = c.smj_prepare(ok, lk)
                sl, sr = plan.expand(0, plan.size)
                plan.release()
            if self.streams > 2:
                lo, ro = fut3.result()
                main.wait_stream(self.s3)
            r1, mask, sel, r6 = fut.result()
            main.wait_stream(self.s2)
            return {"pkfk": (lo, ro), "smj": (sl, sr), "q1": r1, "q6_mask": mask, "q6_sel": sel, "q6": r6}
        self._mark("start")
        if self.exchange:   # shuffled placement: the joins exchange over NCCL
            from paper_2203_01877_b200 import dist
            self.strategy, lo, ro = dist.pkfk_join_shuffled(c, ok, lk, strategy=self.pkfk_strategy, transport=self.transport)
            self._mark("pkfk_join")
            sl, sr = dist.smj_join_copartition(c, ok, lk)
            self._mark("smj_join")
        else:
            lo, ro = c.pkfk_join(ok, lk)
            self._mark("pkfk_join")
            plan = c.smj_prepare(ok, lk)
            sl, sr = plan.expand(0, plan.size)
            plan.release()
            self._mark("smj_join")
        r1 = self.groupby(q1, Q1_KEYS, Q1_AGGS, Q1_PREDS)
        self._mark("q1_groupby")
        mask, sel = c.filter_compact(q6, Q6_PREDS)
        self._mark("q6_filter")
        r6 = self.groupby(q6, [], Q6_AGGS, Q6_PREDS)
        self._mark("q6_sum")
        return {"pkfk": (lo, ro), "smj": (sl, sr), "q1": r1, "q6_mask": mask, "q6_sel": sel, "q6": r6}

    def collect_ops(self):
        torch.cuda.synchronize()
        for i in range(1, len(self._ev)):
            name, e = self._ev[i]
            if name == "start":
                continue
            self.op_ms[name] = self.op_ms.get(name, 0.0) + self._ev[i - 1][1].elapsed_time(e)
        self._ev = []


def run_gpu(args):
    import paper_2203_01877_b200 as T
    rank, world, local = env_rank()
    # test-only overrides: a functional run of the multi-rank code path on a one-GPU box
    # (gloo collectives, every rank on device 0); never used for a reported number
    if os.environ.get("TQP_BENCH_DEVICE") is not None:
        local = int(os.environ["TQP_BENCH_DEVICE"])
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        backend = os.environ.get("TQP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    placement = args.placement or ("exchange" if world > 1 else "local")
    orders, li = make_data(rank, world, dev, args.layout, placement)
    # separate process groups (communicators) for the collectives issued from other threads
    agg_group = ((dist.new_group(list(range(world))), dist.new_group(list(range(world))) if args.streams > 2 else None)
                 if (dist and args.streams > 1) else None)
    hp = HotPath(T, orders, li, world, placement, streams=args.streams, agg_group=agg_group)
    hp.streams = 1   # warm-up, kernel table and per-operator timings: one stream
    hp.transport = args.transport
    hp.pkfk_strategy = args.pkfk_strategy

    def barrier():
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        last = hp.step()
    torch.cuda.synchronize()
    cbytes = compulsory_bytes(hp, last)
    del last
    # Per-kernel table from profiled, untimed steps (two events around every launch
    # cost host time the GPU waits on after each readback, ~0.35 ms per step); the
    # timed region then brackets only the dominant kernel's launches with events.
    prof_steps = 3
    hp.ctx.reset_counters()
    hp.ctx.set_profiling(True)
    for _ in range(prof_steps):
        hp.step()
    ktable = hp.ctx.kernel_stats()
    hp.ctx.set_profiling(False)
    dom_name = max(ktable.items(), key=lambda kv: kv[1][0])[0]
    hp._ev, hp.op_ms = [], {}

    if args.streams > 1:   # per-operator times from sequential steps; the timed steps run concurrently
        for _ in range(2):
            hp.step()
        hp.collect_ops()
        seq_op_ms = {k: v / 2 for k, v in hp.op_ms.items()}
        hp.op_ms = {}
        hp.streams = args.streams
        for _ in range(2):   # warm the concurrent path (second context, worker thread)
            hp.step()
        torch.cuda.synchronize()
    ctxs = [hp.ctx] + ([hp.ctx2] if args.streams > 1 else []) + ([hp.ctx3] if args.streams > 2 else [])

    # ---------------- device-timed region: inputs resident in HBM
    clk = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clk.start()
    for c in ctxs:
        c.reset_counters()
        c.set_profiling(True, only=dom_name)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    from paper_2203_01877_b200 import dist as tdist
    tdist.EXCHANGE_LOG = [] if hp.exchange else None
    t0.record()
    for _ in range(args.steps):
        hp.step()
    t1.record()
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    exchange = None
    if hp.exchange:
        xl, tdist.EXCHANGE_LOG = tdist.EXCHANGE_LOG, None
        x_ms = sum(a.elapsed_time(b) for a, b, _, _ in xl) / args.steps
        x_recv = sum(r for _, _, r, _ in xl) / args.steps
        x_sent = sum(sn for _, _, _, sn in xl) / args.steps
        exchange = {"strategy_pkfk": hp.strategy, "transport": args.transport, "all_to_all_ms_per_step": x_ms,
                    "recv_bytes_per_step": x_recv, "sent_bytes_per_step": x_sent,
                    "nvlink_recv_GBps": x_recv / (x_ms / 1e3) / 1e9 if x_ms > 0 else None,
                    "how": "CUDA events around every all_to_all (NCCL) or fused partition-scatter (p2p) of the step's two "
                           "joins on this rank (rank 0 shown)"}
    ms_local = t0.elapsed_time(t1)
    kstats, launches = {}, 0
    for c in ctxs:   # the dominant kernel may run on either context
        for k, (ms, nl, by) in c.kernel_stats().items():
            a = kstats.get(k, (0.0, 0, 0.0))
            kstats[k] = (a[0] + ms, a[1] + nl, a[2] + by)
        c.set_profiling(False)
        launches += c.launch_count()
    hp.collect_ops()
    op_ms = {k: v / args.steps for k, v in hp.op_ms.items()} if args.streams == 1 else seq_op_ms
    hp.streams = 1
    peak_gbs, _ = peaks()
    operators = {k: {"ms": op_ms[k], "compulsory_bytes": b, "GBps": b / (op_ms[k] / 1e3) / 1e9,
                     "frac_measured_peak": b / (op_ms[k] / 1e3) / 1e9 / peak_gbs,
                     "frac_8TBps": b / (op_ms[k] / 1e3) / 1e9 / 8000.0}
                 for k, b in cbytes.items() if op_ms.get(k)}
    general = general_route_pkfk(hp) if world == 1 else None

    # ---------------- end to end: pinned host inputs -> device -> step -> pinned host results
    host_cols = {"o_orderkey": orders["o_orderkey"]}
    for name in set(Q1_COLS) | set(Q6_COLS) | {"l_orderkey"}:
        host_cols[name] = li[name]
    host = {k: v.cpu().pin_memory() for k, v in host_cols.items()}
    del orders, li
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    pinned_out = {}
    e2e_steps = max(1, min(args.steps, 5))
    d2h = 0

    # Copies overlap compute and each other (PCIe is full duplex): the H2D stream brings
    # the inputs in the order the operators need them (join keys, then Q1's columns,
    # then Q6's), the compute stream waits for each group, and every operator's results
    # go back on a D2H stream as soon as they exist.
    s_cmp = torch.cuda.current_stream(dev)
    s_h2d = torch.cuda.Stream(dev)
    s_d2h = torch.cuda.Stream(dev)
    groups = [["o_orderkey", "l_orderkey"]]
    groups.append([c for c in dict.fromkeys(Q1_COLS) if c not in groups[0]])
    groups.append([c for c in dict.fromkeys(Q6_COLS) if c not in groups[0] + groups[1]])
    slot = [0]

    def to_host(ts):
        ev = torch.cuda.Event()
        ev.record(s_cmp)
        s_d2h.wait_event(ev)
        n = 0
        with torch.cuda.stream(s_d2h):
            for t in ts:
                t.record_stream(s_d2h)
                buf = pinned_out.get(slot[0])
                if buf is None or buf.numel() < t.numel() or buf.dtype != t.dtype:
                    buf = torch.empty(max(t.numel(), 1) * 2, dtype=t.dtype, pin_memory=True)
                    pinned_out[slot[0]] = buf
                buf.view(-1)[:t.numel()].copy_(t.reshape(-1), non_blocking=True)
                n += t.numel() * t.element_size()
                slot[0] += 1
        return n

    def e2e_step():
        slot[0] = 0
        start = torch.cuda.Event()
        start.record(s_cmp)
        s_h2d.wait_event(start)
        dv, ready = {}, []
        with torch.cuda.stream(s_h2d):
            for g in groups:
                for k in g:
                    dv[k] = host[k].to(dev, non_blocking=True)
                    dv[k].record_stream(s_cmp)
                ev = torch.cuda.Event()
                ev.record(s_h2d)
                ready.append(ev)
        c = hp.ctx
        n = 0
        s_cmp.wait_event(ready[0])
        lo, ro = c.pkfk_join(dv["o_orderkey"], dv["l_orderkey"])
        n += to_host([lo, ro])
        plan = c.smj_prepare(dv["o_orderkey"], dv["l_orderkey"])
        sl, sr = plan.expand(0, plan.size)
        plan.release()
        n += to_host([sl, sr])
        s_cmp.wait_event(ready[1])
        r1 = hp.groupby([dv[k] for k in Q1_COLS], Q1_KEYS, Q1_AGGS, Q1_PREDS)
        n += to_host(list(r1["keys"]) + list(r1["results"]))
        s_cmp.wait_event(ready[2])
        q6 = [dv[k] for k in Q6_COLS]
        mask, sel = c.filter_compact(q6, Q6_PREDS)
        n += to_host([mask, sel])
        r6 = hp.groupby(q6, [], Q6_AGGS, Q6_PREDS)
        n += to_host(list(r6["keys"]) + list(r6["results"]))
        done = torch.cuda.Event()
        done.record(s_d2h)
        s_cmp.wait_event(done)
        return n

    e2e_step()
    torch.cuda.synchronize()
    hp._ev = []
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_steps):
        d2h = e2e_step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    hp._ev = []
    e2e_ms_local = e0.elapsed_time(e1) / e2e_steps

    # ---------------- max over ranks
    vals = torch.tensor([ms_local, e2e_ms_local, float(launches)], dtype=torch.float64, device=dev)
    if dist:
        mx = vals.clone()
        dist.all_reduce(mx[:2], op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm[2:], op=dist.ReduceOp.SUM)
        ms_total, e2e_ms, launches_all = float(mx[0]), float(mx[1]), int(sm[2])
    else:
        ms_total, e2e_ms, launches_all = ms_local, e2e_ms_local, launches
    ms_step = ms_total / args.steps
    rows_total = hp.n * world      # identical partition sizes are not guaranteed: use the sum
    if dist:
        t = torch.tensor([float(hp.n)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        rows_total = float(t)
    value = rows_total / (ms_step / 1e3)

    if rank == 0:
        peak, peak_src = peaks()
        name = dom_name
        kms, klaunch, kbytes = kstats[name]
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(name)
        achieved = (kbytes / klaunch) / (kms / klaunch / 1e3) / 1e9 if kms > 0 else 0.0
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "rows/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int64",
            "data": f"synthetic (in-repo TPC-H-shaped generator, seed {SEED}; dbgen unavailable offline)",
            "config": {
                "workload": f"tpch_sf{SF_PER_RANK:g}_hot_path: pkfk_join + smj_join(orders x lineitem) + Q1 groupby + "
                            "Q6 filter/sum",
                "sf_per_rank": SF_PER_RANK,
                "lineitem_rows_per_rank": hp.n,
                "orders_rows_per_rank": hp.ok.numel(),
                "layout": f"lineitem rows {args.layout}",
                "placement": (placement + (": every rank's lineitem references orders on every rank; the "
                              "joins exchange (key, global row) over NCCL" if placement == "exchange" else
                              ": each rank's lineitem references only its own orders (no join exchange)")),
                "parallelism": f"dp{world}",
                "streams": args.streams,
                "concurrency": ({1: "one stream, operators in sequence",
                                 2: "timed steps: the aggregation queries (Q1, Q6 filter, Q6 sum) on a second CUDA stream "
                                    "with their own libtqp context, concurrently with the joins",
                                 3: "timed steps: the aggregation queries, the PK-FK join and the SMJ on three CUDA "
                                    "streams with their own libtqp contexts, concurrently"}[args.streams] +
                                ("; per-operator times and the kernel table from sequential steps" if args.streams > 1 else "")),
                "l2": "inputs larger than L2: 2.8 GB of columns per rank per step vs 126 MB L2 (no flush needed)",
            },
            "clocks": clocks,
            "e2e": {"value": rows_total / (e2e_ms / 1e3), "unit": "rows/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                    "how": "pinned host columns -> H2D -> same step via the public API -> D2H of every result; "
                           "H2D, compute and D2H on three streams, each operator's inputs awaited and its "
                           "results copied out as soon as they exist"},
            "gpu_launches": launches_all,
            "roofline": {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": kbytes / max(klaunch, 1),
                         "avg_launch_ms": kms / max(klaunch, 1), "launches": klaunch,
                         "share_of_step": kms / ms_total if ms_total else None},
            "operators_ms": op_ms,
            "operators": operators,
            "operators_how": "per-operator CUDA events inside the timed steps; compulsory bytes per SURVEY.md "
                             "§8(d) (sort 24 B/key, index pairs 16 B, columns read once); frac against the "
                             "measured copy peak and against 8 TB/s",
            "pkfk_general_route": general,
            "probe_rows_per_s": hp.n / (op_ms.get("pkfk_join", float("nan")) / 1e3),
            "groupby_rows_per_s": hp.n / (op_ms.get("q1_groupby", float("nan")) / 1e3),
            "kernels_how": f"every launch bracketed by events over {prof_steps} untimed steps "
                           "(the timed region brackets only the dominant kernel)",
            "kernels": {k: {"ms_per_step": v[0] / prof_steps, "launches_per_step": v[1] / prof_steps,
                            "algorithmic_GBps": (v[2] / v[0] / 1e6) if v[0] > 0 else None}
                        for k, v in sorted(ktable.items(), key=lambda kv: -kv[1][0])},
        }
        if exchange is not None:
            line["exchange"] = exchange
        if not args.no_cpu_baseline and world == 1:   # the oracle baseline: rank 0 at N = 1 only
            line["cpu_baseline"] = cpu_baseline(hp, args)
        if world == 1 and not args.no_sf100:
            del hp
            line["sf100"] = sf100_ops(T, dev, peak_gbs)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _timed(f, reps):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def general_route_pkfk(hp, reps=5):
    """The PK-FK join when the build side is NOT already in key order (orders shuffled by a
    seeded permutation, made outside the timed region): the radix-sorted build side and
    the slot-table probe instead of the presorted rank-bitmap route of the main step."""
    g = torch.Generator(device=hp.ok.device).manual_seed(7)
    ok_shuf = hp.ok[torch.randperm(hp.ok.numel(), device=hp.ok.device, generator=g)]
    ms = _timed(lambda: hp.ctx.pkfk_join(ok_shuf, hp.lk), reps)
    nb, npr = ok_shuf.numel(), hp.lk.numel()
    b = 24 * nb + 8 * nb + 8 * npr + 16 * npr
    out = {"ms": ms, "compulsory_bytes": b, "GBps": b / (ms / 1e3) / 1e9, "probe_rows_per_s": npr / (ms / 1e3),
           "how": "orders keys permuted (seed 7) outside the timing; median-free mean of 5 calls, CUDA events"}
    del ok_shuf
    return out


def sf100_ops(T, dev, peak_gbs, reps=3):
    """SF100 on one GPU (BASELINE configs[4]'s per-GPU size at N = 1; the north-star target
    operators): PK-FK join (150M orders x ~600M lineitem) and Q1, CUDA events around each
    call, after one untimed call."""
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    orders, li = tpch_orders_lineitem(100.0, seed=42, device=dev, layout="shuffled")
    ok, lk = orders["o_orderkey"], li["l_orderkey"]
    q1 = columns(li, Q1_COLS)
    keep = set(Q1_COLS) | {"l_orderkey"}
    for k in list(li):
        if k not in keep:
            del li[k]
    ctx = T.context()
    res = {}
    ms = _timed(lambda: ctx.pkfk_join(ok, lk), reps)
    nb, npr = ok.numel(), lk.numel()
    b = 24 * nb + 8 * nb + 8 * npr + 16 * npr
    res["pkfk_join"] = {"ms": ms, "compulsory_bytes": b, "GBps": b / (ms / 1e3) / 1e9,
                        "frac_measured_peak": b / (ms / 1e3) / 1e9 / peak_gbs, "probe_rows_per_s": npr / (ms / 1e3)}
    ms = _timed(lambda: ctx.groupby_agg(q1, Q1_KEYS, Q1_AGGS, Q1_PREDS), reps)
    b = sum(c.element_size() for c in q1) * npr
    res["q1_groupby"] = {"ms": ms, "compulsory_bytes": b, "GBps": b / (ms / 1e3) / 1e9,
                         "frac_measured_peak": b / (ms / 1e3) / 1e9 / peak_gbs, "rows_per_s": npr / (ms / 1e3)}
    res["rows"] = {"orders": nb, "lineitem": npr}
    del orders, li, ok, lk, q1
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------ CPU oracle leg

def oracle_sample(orders, li, sf_sample):
    """A bounded sample of the same workload: the first orders rows and their lineitems."""
    n_s = orders_count(sf_sample)
    m = li["l_parent"] < n_s
    ok = orders["o_orderkey"][:n_s].cpu().numpy()
    lcols = {k: v[m].cpu().numpy().astype(np.int64) for k, v in li.items()
             if k in set(Q1_COLS) | set(Q6_COLS) | {"l_orderkey"}}
    return ok, lcols


def oracle_step(ok, lc):
    import oracle
    oracle.pkfk_join(ok, lc["l_orderkey"])
    oracle.smj_join(ok, lc["l_orderkey"])
    oracle.groupby_agg([lc[c] for c in Q1_COLS], Q1_KEYS, Q1_AGGS, Q1_PREDS)
    oracle.filter_compact([lc[c] for c in Q6_COLS], Q6_PREDS)
    oracle.groupby_agg([lc[c] for c in Q6_COLS], [], Q6_AGGS, Q6_PREDS)


def cpu_baseline(hp, args):
    """The oracle as it stands (single-threaded C), rank 0 only, bounded sample."""
    sfs = args.cpu_sample_sf
    orders = {"o_orderkey": hp.ok}
    li = {"l_orderkey": hp.lk, **{c: t for c, t in zip(Q1_COLS, hp.q1)}, **{c: t for c, t in zip(Q6_COLS, hp.q6)}}
    # l_parent is needed for the sample mask: rebuild it from the generator (bookkeeping, not method)
    _, li_full = tpch_orders_lineitem(sfs, seed=42, device="cpu", layout="shuffled")
    orders_s, _ = tpch_orders_lineitem(sfs, seed=42, device="cpu", layout="shuffled")
    ok = orders_s["o_orderkey"].numpy()
    lc = {k: v.numpy().astype(np.int64) for k, v in li_full.items()
          if k in set(Q1_COLS) | set(Q6_COLS) | {"l_orderkey"}}
    del orders, li
    t0 = time.perf_counter()
    oracle_step(ok, lc)
    one = time.perf_counter() - t0
    reps = max(1, min(int(20.0 // max(one, 1e-3)), 5))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle_step(ok, lc)
    dt = (time.perf_counter() - t0) / reps
    n = lc["l_orderkey"].size
    return {"value": n / dt, "unit": "rows/s", "cores": 1, "kind": "oracle",
            "sample": f"TPC-H-shaped SF{sfs} ({n} lineitem rows, same generator/queries), "
                      f"{reps} timed oracle steps after 1 untimed, host cores available: {os.cpu_count()}",
            "ms_per_step": dt * 1e3}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    sfs = args.cpu_sample_sf
    orders, li = tpch_orders_lineitem(sfs, seed=42, device="cpu", layout="shuffled")
    ok = orders["o_orderkey"].numpy()
    lc = {k: v.numpy().astype(np.int64) for k, v in li.items() if k in set(Q1_COLS) | set(Q6_COLS) | {"l_orderkey"}}
    for _ in range(args.warmup):
        oracle_step(ok, lc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(ok, lc)
    dt = (time.perf_counter() - t0) / args.steps
    n = lc["l_orderkey"].size
    v = n / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (in-repo TPC-H-shaped generator, seed 42)",
        "config": {"workload": "tpch_sf10_hot_path: pkfk_join + smj_join(orders x lineitem) + Q1 groupby + "
                               "Q6 filter/sum", "sample_sf": sfs,
                   "sample": f"each step runs the workload's operators on a bounded SF{sfs} sample "
                             f"({n} lineitem rows), not the SF{SF_PER_RANK:g} batch",
                   "parallelism": "host oracle, 1 core"},
        "cpu_baseline": {"value": v, "unit": "rows/s", "cores": 1, "kind": "oracle",
                         "sample": f"TPC-H-shaped SF{sfs} ({n} lineitem rows) per step; single-threaded C oracle"},
        "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    # tqp: this library; reference: the oracle on host cores (the driver's reference arm);
    # paper-torch: the paper's tensor programs as torch ops on the same GPU (comparison only)
    ap.add_argument("--impl", default="tqp", choices=["tqp", "reference", "paper-torch"])
    ap.add_argument("--layout", default="shuffled", choices=["shuffled", "clustered"])
    # N > 1: exchange (default) = lineitem's orders spread over all ranks, joins exchange over
    # NCCL; local = each rank's lineitem joins only its own orders
    ap.add_argument("--placement", default=None, choices=["exchange", "local"])
    ap.add_argument("--no-sf100", action="store_true", help="skip the SF100 single-GPU operator section")
    # 2: the aggregation queries run on a second stream concurrently with the joins in the
    # timed steps (per-operator times always come from sequential steps)
    ap.add_argument("--streams", type=int, default=2, choices=[1, 2, 3])
    # N > 1, co-partitioned PK-FK join: NCCL all_to_all, or the fused partition kernel storing
    # straight into the peers' receive buffers (CUDA IPC / NVLink P2P)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"])
    ap.add_argument("--pkfk-strategy", default="auto", choices=["auto", "broadcast", "copartition"])
    ap.add_argument("--cpu-sample-sf", type=float, default=0.25)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # the workload: TPC-H scale factor per rank (BASELINE.json's metric is quoted at 10) and
    # the generator seed
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=42)
    args = ap.parse_args()
    global SF_PER_RANK, SEED
    SF_PER_RANK, SEED = args.sf, args.seed
    if args.warmup < 3 and args.impl == "tqp":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    if args.impl == "paper-torch":
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
        import paper_torch
        print(json.dumps(paper_torch.run(max(args.steps, 1), max(args.warmup, 1), check=True)))
        return 0
    run_gpu(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
