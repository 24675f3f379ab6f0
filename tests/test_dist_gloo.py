"""World-size-2 gloo tests (CPU) of the multi-GPU exchange logic in
paper_2203_01877_b200/dist.py. The local operators are the oracle (CPU), so the
test checks the partitioning, all-gather, AVG rewrite and exact merge, and the
broadcast-build join's global row numbering against the single-process oracle
on the whole table."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---- oracle-backed stand-ins for the CUDA operators (same dict layout as the binding)

def oracle_local(cols, key_idx, aggs, preds):
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


def oracle_merge(keys, aggs, partials, counts):
    """Plain merge by dictionary (Python big ints) -- mirrors tqp_groupby_merge's contract."""
    m = counts.numel()
    groups = {}
    for i in range(m):
        k = tuple(int(t[i]) for t in keys)
        g = groups.setdefault(k, {"count": 0, "vals": [None] * len(aggs)})
        g["count"] += int(counts[i])
        for a, (op, _) in enumerate(aggs):
            p = partials[a]
            if op in ("sum", "avg"):
                lo, hi = int(p[i, 0]) & ((1 << 64) - 1), int(p[i, 1])
                v = (hi << 64) + lo
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


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from datagen import tpch_orders_lineitem
        from datagen.tpch import orders_count
        from datagen.queries import Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS, Q6_AGGS, Q6_COLS, Q6_PREDS, columns
        from paper_2203_01877_b200 import dist as D   # noqa: imports the binding (CPU: no kernels run)
        sf = 0.01
        n_o = orders_count(sf) // world
        orders, li = tpch_orders_lineitem(sf, seed=42, device="cpu", layout="shuffled",
                                          order_range=(rank * n_o, (rank + 1) * n_o))
        q1 = D.groupby_agg(None, columns(li, Q1_COLS), Q1_KEYS, Q1_AGGS, Q1_PREDS,
                           local_fn=oracle_local, merge_fn=oracle_merge)
        q6 = D.groupby_agg(None, columns(li, Q6_COLS), [], Q6_AGGS, Q6_PREDS,
                           local_fn=oracle_local, merge_fn=oracle_merge)
        # shuffled layout: each rank probes with a different lineitem slice than its orders
        import oracle
        def join_fn(b, p):
            lo, ro = oracle.pkfk_join(b.numpy(), p.numpy())
            return torch.as_tensor(lo), torch.as_tensor(ro)
        other = (rank + 1) % world
        _, li_other = tpch_orders_lineitem(sf, seed=42, device="cpu", layout="shuffled",
                                           order_range=(other * n_o, (other + 1) * n_o))
        lo, ro = D.pkfk_join_broadcast(None, orders["o_orderkey"], li_other["l_orderkey"], join_fn=join_fn)
        out_q.put((rank, q1, q6, lo.numpy(), ro.numpy(), li_other["l_parent"].numpy() + other * n_o))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_groupby_and_broadcast_join():
    import oracle
    from datagen import tpch_orders_lineitem
    from datagen.queries import Q1_AGGS, Q1_COLS, Q1_KEYS, Q1_PREDS, Q6_AGGS, Q6_COLS, Q6_PREDS, columns
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # single-process oracle over the whole table (the union of both ranks' slices)
    sf = 0.01
    _, full = tpch_orders_lineitem(sf, seed=42, device="cpu", layout="shuffled")
    want1 = oracle.groupby_agg([c.numpy() for c in columns(full, Q1_COLS)], Q1_KEYS, Q1_AGGS, Q1_PREDS)
    want6 = oracle.groupby_agg([c.numpy() for c in columns(full, Q6_COLS)], [], Q6_AGGS, Q6_PREDS)
    for rank, q1, q6, lo, ro, parent_global in outs:
        assert q1["n_groups"] == want1["n_groups"]
        assert [list(map(int, k)) for k in q1["keys"]] == [k.tolist() for k in want1["keys"]]
        for a, (op, _) in enumerate(Q1_AGGS):
            if op == "avg":
                assert np.allclose(q1["results"][a], want1["results"][a], rtol=1e-12, atol=0)
            else:
                assert q1["results"][a] == want1["results"][a]
        assert q6["results"][0] == want6["results"][0]
        # broadcast build: global orders row of every probed lineitem, probe-row order
        assert np.array_equal(ro, np.arange(len(ro)))
        assert np.array_equal(lo, parent_global)


def _worker_copart(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from datagen import tpch_orders_lineitem
        from datagen.tpch import orders_count
        from paper_2203_01877_b200 import dist as D
        sf = 0.01
        n_o = orders_count(sf) // world
        orders, _ = tpch_orders_lineitem(sf, seed=42, device="cpu", layout="shuffled",
                                         order_range=(rank * n_o, (rank + 1) * n_o))
        other = (rank + 1) % world   # shuffled layout: the probe slice belongs to another rank's orders
        _, li = tpch_orders_lineitem(sf, seed=42, device="cpu", layout="shuffled",
                                     order_range=(other * n_o, (other + 1) * n_o))

        def join_fn(b, p):
            lo, ro = oracle.pkfk_join(b.numpy(), p.numpy())
            return torch.as_tensor(lo), torch.as_tensor(ro)

        res = {}
        for strategy in ("copartition", "broadcast", "auto"):
            s, gl, gr = D.pkfk_join_shuffled(None, orders["o_orderkey"], orders["o_global_row"], li["l_orderkey"],
                                             li["l_global_row"], strategy=strategy, join_fn=join_fn)
            res[strategy] = (s, gl.numpy(), gr.numpy())
        parent_global = li["l_parent"].numpy() + other * n_o
        out_q.put((rank, res, li["l_global_row"].numpy(), parent_global,
                   D.pkfk_cost_bytes(orders_count(sf), 0, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_copartition_join_and_cost_model():
    """Co-partitioned shuffled-layout PK-FK join: the union over ranks of (global build
    row, global probe row), ordered by probe row, is the single-process join of the whole
    table; broadcast gives the same pairs; 'auto' takes the cheaper exchange."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_copart, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # expected: every lineitem row joins its parent order (generator closed form)
    rows = np.concatenate([o[2] for o in outs])
    parents = np.concatenate([o[3] for o in outs])
    order = np.argsort(rows, kind="stable")
    want_l, want_r = parents[order], rows[order]
    gl = np.concatenate([o[1]["copartition"][1] for o in outs])
    gr = np.concatenate([o[1]["copartition"][2] for o in outs])
    o2 = np.argsort(gr, kind="stable")
    assert np.array_equal(gr[o2], want_r) and np.array_equal(gl[o2], want_l)
    for rank, res, *_ in outs:   # within a rank, co-partition pairs ascend by global probe row
        assert np.all(np.diff(res["copartition"][2]) > 0)
    bl = np.concatenate([o[1]["broadcast"][1] for o in outs])
    br = np.concatenate([o[1]["broadcast"][2] for o in outs])
    o3 = np.argsort(br, kind="stable")
    assert np.array_equal(br[o3], want_r) and np.array_equal(bl[o3], want_l)
    for _, res, *_ in outs:
        s = res["auto"][0]
        n_b, n_p = 15_000, len(rows)
        cost = {"broadcast": n_b * 8 * 0.5, "copartition": (n_b + n_p) / 2 * 16 * 0.5}
        assert s == min(cost, key=cost.get)


def _skewed(n, seed):
    """Keys in [0, 400) with key 7 on about a quarter of the rows (a Zipf-like heavy key)."""
    g = torch.Generator().manual_seed(seed)
    k = torch.randint(0, 400, (n,), generator=g, dtype=torch.int64)
    k[torch.rand(n, generator=g) < 0.25] = 7
    return k


def _worker_sort_smj(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from datagen import uniform_keys, zipf_keys
        from paper_2203_01877_b200 import dist as D

        def sort_fn(k):
            s, p = oracle.sort(k.numpy())
            return torch.as_tensor(s), torch.as_tensor(p)

        def join_fn(a, b):
            lo, ro = oracle.smj_join(a.numpy(), b.numpy())
            return torch.as_tensor(lo), torch.as_tensor(ro)

        n = 20_000
        keys = zipf_keys(world * n, 5_000, seed=42)            # global column, Zipf with duplicates
        mine = keys[rank * n:(rank + 1) * n]
        rows = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int64)
        sk, sr = D.sort_samplesort(None, mine, rows, sort_fn=sort_fn)
        left = zipf_keys(world * n, 3_000, seed=7)
        right = uniform_keys(world * n, 3_000, seed=8)
        sl = left[rank * n:(rank + 1) * n]
        sr2 = right[rank * n:(rank + 1) * n]
        gl, gr = D.smj_join_copartition(None, sl, rows, sr2, rows, join_fn=join_fn, sort_fn=None)
        # skewed: one key holds ~25 % of each side (spans both ranks' key ranges)
        m = 3_000
        hl, hr = _skewed(world * m, 11), _skewed(world * m, 12)
        hrows = torch.arange(rank * m, (rank + 1) * m, dtype=torch.int64)
        hl_, hr_ = D.smj_join_copartition(None, hl[rank * m:(rank + 1) * m], hrows, hr[rank * m:(rank + 1) * m],
                                          hrows, join_fn=join_fn, sort_fn=None)
        out_q.put((rank, sk.numpy(), sr.numpy(), gl.numpy(), gr.numpy(), hl_.numpy(), hr_.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_samplesort_and_smj():
    """Distributed sample sort and co-partitioned SMJ: the ranks' outputs concatenated in
    rank order equal the single-process stable sort / Alg.-1 join of the whole columns."""
    import oracle
    from datagen import uniform_keys, zipf_keys
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sort_smj, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    n = 20_000
    keys = zipf_keys(world * n, 5_000, seed=42).numpy()
    want_k, want_p = oracle.sort(keys)
    assert np.array_equal(np.concatenate([o[1] for o in outs]), want_k)
    assert np.array_equal(np.concatenate([o[2] for o in outs]), want_p)
    left = zipf_keys(world * n, 3_000, seed=7).numpy()
    right = uniform_keys(world * n, 3_000, seed=8).numpy()
    # skewed case: exact single-process order, and the heavy key's pairs split over the ranks
    m = 3_000
    hl, hr = _skewed(world * m, 11).numpy(), _skewed(world * m, 12).numpy()
    wl, wr = oracle.smj_join(hl, hr)
    assert np.array_equal(np.concatenate([o[5] for o in outs]), wl)
    assert np.array_equal(np.concatenate([o[6] for o in outs]), wr)
    heavy = [int((hl[o[5]] == 7).sum()) for o in outs]
    assert min(heavy) > 0.25 * sum(heavy), heavy
    olo, oro = oracle.smj_join(left, right)
    assert np.array_equal(np.concatenate([o[3] for o in outs]), olo)
    assert np.array_equal(np.concatenate([o[4] for o in outs]), oro)
