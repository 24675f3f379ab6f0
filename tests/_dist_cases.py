"""Multi-rank cases of paper_2203_01877_b200/dist.py shared by the CPU (gloo, oracle-backed
local operators) and GPU (gloo with host staging, libtqp local operators on one GPU)
tests. Not a test module itself.

Every rank holds a slice of each column; the expected results are the single-process
oracle over the rank-ordered concatenation of the slices ("global row" = position in
that concatenation, the contract of dist.py)."""

import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SF = 0.01


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------- oracle-backed local operators (CPU)

class OracleOps:
    """CPU stand-ins for the libtqp context methods dist.py calls (test infrastructure:
    the oracle for the operators, numpy for the partition / gather plumbing)."""

    def sort(self, keys):
        import oracle
        s, p = oracle.sort(keys.numpy())
        return torch.as_tensor(s).to(keys.dtype), torch.as_tensor(p)

    def pkfk_join(self, b, p):
        import oracle
        lo, ro = oracle.pkfk_join(b.numpy(), p.numpy())
        return torch.as_tensor(lo), torch.as_tensor(ro)

    def pkfk_join_payload(self, b, p, bpay, ppay, indices=False):
        lo, ro = self.pkfk_join(b, p)
        return [c[lo] for c in bpay], [c[ro] for c in ppay], ((lo, ro) if indices else None)

    def smj_join_payload(self, l, r, lpay, rpay, indices=False):
        import oracle
        lo, ro = oracle.smj_join(l.numpy(), r.numpy())
        lo, ro = torch.as_tensor(lo), torch.as_tensor(ro)
        return [c[lo] for c in lpay], [c[ro] for c in rpay], ((lo, ro) if indices else None)

    def partition(self, keys, splitters, row_base=0, rows=True):
        k = keys.numpy().astype(np.int64)
        dest = np.searchsorted(splitters.numpy(), k, side="right")
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=splitters.numel() + 1)
        return (keys[torch.as_tensor(order)], torch.as_tensor(order + row_base) if rows else None,
                torch.as_tensor(counts, dtype=torch.int64))

    def minmax(self, keys):
        if keys.numel() == 0:
            return torch.tensor([np.iinfo(np.int64).max, np.iinfo(np.int64).min], dtype=torch.int64)
        return torch.tensor([int(keys.min()), int(keys.max())], dtype=torch.int64)

    def range_splitters(self, lohi, parts):
        lo, hi = int(lohi[0]), int(lohi[1])
        w = (hi - lo) // parts + 1
        return torch.tensor([min(lo + (j + 1) * w, np.iinfo(np.int64).max) for j in range(parts - 1)],
                            dtype=torch.int64)

    def gather(self, src, idx):
        return src[idx]

    def groupby_agg(self, cols, key_idx, aggs, preds):
        import oracle
        r = oracle.groupby_agg([c.numpy() for c in cols], key_idx, aggs, preds)
        G = r["n_groups"]
        res = []
        for (op, _), v in zip(aggs, r["results"]):
            if op == "sum":
                res.append(torch.tensor([[x & ((1 << 64) - 1) if x & ((1 << 64) - 1) < (1 << 63)
                                          else (x & ((1 << 64) - 1)) - (1 << 64), x >> 64] for x in v],
                                        dtype=torch.int64).reshape(G, 2))
            elif op == "avg":
                res.append(torch.tensor(v, dtype=torch.float64))
            else:
                res.append(torch.tensor(v, dtype=torch.int64))
        keys = [torch.tensor(k, dtype=cols[key_idx[i]].dtype) for i, k in enumerate(r["keys"])]
        return {"n_groups": G, "keys": keys, "results": res}

    def groupby_merge(self, keys, aggs, partials, counts):
        """Plain merge by dictionary (Python big ints) -- tqp_groupby_merge's contract."""
        groups = {}
        for i in range(counts.numel()):
            k = tuple(int(t[i]) for t in keys)
            g = groups.setdefault(k, {"count": 0, "vals": [None] * len(aggs)})
            g["count"] += int(counts[i])
            for a, (op, _) in enumerate(aggs):
                p = partials[a]
                if op in ("sum", "avg"):
                    v = (int(p[i, 1]) << 64) + (int(p[i, 0]) & ((1 << 64) - 1))
                    g["vals"][a] = v if g["vals"][a] is None else g["vals"][a] + v
                elif op == "min":
                    g["vals"][a] = int(p[i]) if g["vals"][a] is None else min(g["vals"][a], int(p[i]))
                elif op == "max":
                    g["vals"][a] = int(p[i]) if g["vals"][a] is None else max(g["vals"][a], int(p[i]))
        out_keys = sorted(groups)
        results = []
        for a, (op, _) in enumerate(aggs):
            col = []
            for k in out_keys:
                g = groups[k]
                if op == "count":
                    col.append(g["count"])
                elif op == "avg":
                    col.append(float(g["vals"][a]) / g["count"] if g["count"] else float("nan"))
                else:
                    col.append(g["vals"][a])
            results.append(col)
        return {"n_groups": len(out_keys), "keys": [[k[j] for k in out_keys] for j in range(len(keys))],
                "results": results}


# ------------------------------------------------------------------------- inputs

def rank_tables(rank, world, device):
    """Rank's orders slice and its lineitem slice re-parented over every rank's orders
    (datagen.spread_orderkeys): the shuffled multi-rank layout."""
    from datagen import tpch_orders_lineitem
    from datagen.tpch import orders_count, spread_orderkeys
    n_o = orders_count(SF) // world
    orders, li = tpch_orders_lineitem(SF, seed=42, device=device, layout="shuffled",
                                      order_range=(rank * n_o, (rank + 1) * n_o))
    lk, parent = spread_orderkeys(li["l_parent"], rank, world)
    return orders, li, lk, parent


def skewed(n, seed):
    """Keys in [0, 400) with key 7 on about a quarter of the rows (a Zipf-like heavy key)."""
    g = torch.Generator().manual_seed(seed)
    k = torch.randint(0, 400, (n,), generator=g, dtype=torch.int64)
    k[torch.rand(n, generator=g) < 0.25] = 7
    return k


def smj_inputs(world):
    from datagen import uniform_keys, zipf_keys
    n = 20_000
    return {"zipf": (zipf_keys(world * n, 3_000, seed=7), uniform_keys(world * n, 3_000, seed=8)),
            "skewed": (skewed(world * 3_000, 11), skewed(world * 3_000, 12)),
            "sortkeys": zipf_keys(world * n, 5_000, seed=42)}


def _slice(t, rank, world):
    n = t.numel() // world
    hi = (rank + 1) * n if rank + 1 < world else t.numel()
    return t[rank * n:hi]


# ------------------------------------------------------------------------- worker

def worker(rank, world, port, use_gpu, out_q, transport="nccl"):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from datagen.queries import Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS, Q6_AGGS, Q6_COLS, Q6_PREDS, columns
        from paper_2203_01877_b200 import dist as D
        if use_gpu:
            import paper_2203_01877_b200 as T
            torch.cuda.set_device(0)
            ops, dev = T.context(), "cuda"
        else:
            ops, dev = OracleOps(), "cpu"
        h = lambda t: t.cpu().numpy()   # noqa: E731
        out = {"rank": rank}
        orders, li, lk, parent = rank_tables(rank, world, dev)
        # group-by: Q1 / Q6 over the rank's lineitem rows
        q1 = D.groupby_agg(ops, columns(li, Q1_COLS), Q1_KEYS, Q1_AGGS, Q1_PREDS)
        q6 = D.groupby_agg(ops, columns(li, Q6_COLS), [], Q6_AGGS, Q6_PREDS)
        if use_gpu:
            conv = lambda r: {"n_groups": r["n_groups"], "keys": [h(k).tolist() for k in r["keys"]],   # noqa: E731
                              "results": [T.int128_to_ints(x) if x.dim() == 2 else h(x).tolist() for x in r["results"]]}
            q1, q6 = conv(q1), conv(q6)
        out["q1"], out["q6"] = q1, q6
        # PK-FK join, shuffled layout, both exchanges
        for strategy in ("copartition", "broadcast", "auto"):
            ex = {}
            s, gl, gr = D.pkfk_join_shuffled(ops, orders["o_orderkey"], lk, strategy=strategy, exchange=ex,
                                             transport=transport)
            out["pkfk_" + strategy] = (s, h(gl), h(gr), ex)
        if transport == "p2p":   # twice more: the arenas are reused (and grow once for the int32 case)
            for _ in range(2):
                s, gl, gr = D.pkfk_join_shuffled(ops, orders["o_orderkey"], lk, strategy="copartition",
                                                 transport=transport)
                assert (h(gl) == out["pkfk_copartition"][1]).all() and (h(gr) == out["pkfk_copartition"][2]).all()
        out["parent"] = h(parent)
        # int32 keys through the partition (co-partition) path
        s, gl, gr = D.pkfk_join_shuffled(ops, orders["o_orderkey"].to(torch.int32), lk.to(torch.int32),
                                         strategy="copartition", transport=transport)
        out["pkfk_i32"] = (h(gl), h(gr))
        # sample sort and SMJ on slices of global columns
        inp = smj_inputs(world)
        sk, srows = D.sort_samplesort(ops, _slice(inp["sortkeys"], rank, world).to(dev))
        out["sort"] = (h(sk), h(srows))
        for name in ("zipf", "skewed"):
            l, r = inp[name]
            gl, gr = D.smj_join_copartition(ops, _slice(l, rank, world).to(dev), _slice(r, rank, world).to(dev))
            out["smj_" + name] = (h(gl), h(gr))
        # fp64 aggregates are rejected by the distributed group-by
        try:
            D.groupby_agg(ops, [li["l_quantity"].to(torch.float64)], [], [("sum", [(0, 0, 1)])])
            out["f64_rejected"] = False
        except ValueError:
            out["f64_rejected"] = True
        out_q.put(out)
    finally:
        dist.destroy_process_group()


def run(world, use_gpu, transport="nccl"):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, use_gpu, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=600) for _ in range(world)], key=lambda o: o["rank"])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return outs


# ------------------------------------------------------------------------- checks

def check(outs, world):
    import oracle
    from datagen.queries import Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS, Q6_AGGS, Q6_COLS, Q6_PREDS, columns
    tabs = [rank_tables(r, world, "cpu") for r in range(world)]
    li_cat = {k: torch.cat([t[1][k] for t in tabs]) for k in tabs[0][1]}
    bk = torch.cat([t[0]["o_orderkey"] for t in tabs]).numpy()
    pk = torch.cat([t[2] for t in tabs]).numpy()
    # group-by: every rank holds the merged result of the whole table
    want1 = oracle.groupby_agg([c.numpy() for c in columns(li_cat, Q1_COLS)], Q1_KEYS, Q1_AGGS, Q1_PREDS)
    want6 = oracle.groupby_agg([c.numpy() for c in columns(li_cat, Q6_COLS)], [], Q6_AGGS, Q6_PREDS)
    for o in outs:
        q1 = o["q1"]
        assert q1["n_groups"] == want1["n_groups"]
        assert [list(map(int, k)) for k in q1["keys"]] == [list(map(int, k)) for k in want1["keys"]]
        for a, (op, _) in enumerate(Q1_AGGS):
            if op == "avg":
                assert np.allclose(q1["results"][a], want1["results"][a], rtol=1e-12, atol=0)
            else:
                assert list(q1["results"][a]) == list(want1["results"][a])
        assert list(o["q6"]["results"][0]) == list(want6["results"][0])
        assert o["f64_rejected"]
    # PK-FK: the single-process join of the concatenated tables; closed form: parent rows
    wl, wr = oracle.pkfk_join(bk, pk)
    assert np.array_equal(wr, np.arange(len(pk)))
    assert np.array_equal(wl, np.concatenate([o["parent"] for o in outs]))
    for key in ("pkfk_copartition", "pkfk_broadcast", "pkfk_auto"):
        gl = np.concatenate([o[key][1] for o in outs])
        gr = np.concatenate([o[key][2] for o in outs])
        for o in outs:   # within a rank, pairs ascend by global probe row
            assert np.all(np.diff(o[key][2]) > 0)
        order = np.argsort(gr, kind="stable")
        assert np.array_equal(gr[order], wr) and np.array_equal(gl[order], wl), key
    if world > 1:   # co-partition moved rows; byte accounting present
        assert sum(o["pkfk_copartition"][3]["recv_bytes"] for o in outs) > 0
    nb, np_ = len(bk), len(pk)
    cost = {"broadcast": nb * 8 * (world - 1) / world, "copartition": (nb + np_) / world * 16 * (world - 1) / world}
    for o in outs:
        assert o["pkfk_auto"][0] == min(cost, key=cost.get)
    gl = np.concatenate([o["pkfk_i32"][0] for o in outs])
    gr = np.concatenate([o["pkfk_i32"][1] for o in outs])
    order = np.argsort(gr, kind="stable")
    assert np.array_equal(gr[order], wr) and np.array_equal(gl[order], wl)
    # sample sort: concatenation in rank order = the stable sort of the concatenated column
    inp = smj_inputs(world)
    keys = torch.cat([_slice(inp["sortkeys"], r, world) for r in range(world)]).numpy()
    ws, wp = oracle.sort(keys)
    assert np.array_equal(np.concatenate([o["sort"][0] for o in outs]), ws)
    assert np.array_equal(np.concatenate([o["sort"][1] for o in outs]), wp)
    # SMJ: concatenation in rank order = Alg. 1's (key, l, r) order on the whole columns
    for name in ("zipf", "skewed"):
        l, r = inp[name]
        l = torch.cat([_slice(l, q, world) for q in range(world)]).numpy()
        r = torch.cat([_slice(r, q, world) for q in range(world)]).numpy()
        ol, orr = oracle.smj_join(l, r)
        assert np.array_equal(np.concatenate([o["smj_" + name][0] for o in outs]), ol), name
        assert np.array_equal(np.concatenate([o["smj_" + name][1] for o in outs]), orr), name
        if name == "skewed" and world > 1:   # the heavy key's pairs are split over the ranks
            heavy = [int((l[o["smj_skewed"][0]] == 7).sum()) for o in outs]
            assert min(heavy) > 0.25 * sum(heavy), heavy
