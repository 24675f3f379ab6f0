"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL) for the exchanges.

The hot path shards by row ranges (the paper lists data-parallel
execution as future work):
  * group-by: every rank aggregates its rows (tqp_groupby_agg) with AVG rewritten as
    SUM + COUNT; the few partial groups are all-gathered and merged exactly by
    tqp_groupby_merge (int128 sums, averages recomputed from merged SUM / COUNT, never
    averaged);
  * PK-FK join, co-partitioned layout (each rank holds its orders and exactly their
    lineitems): purely local, no exchange;
  * PK-FK join, shuffled layout: the build side is all-gathered (broadcast build,
    SURVEY.md §8(e)); the gathered rank-ordered concatenation is the global build table,
    so build rows come out as global row numbers with no extra remapping.
Operators are injectable (`local_fn`, `merge_fn`, `join_fn`) so the exchange logic is
tested on CPU with the gloo backend and the oracle as the local operator
(tests/test_dist_gloo.py). The product path always uses the libtqp kernels.
"""

import torch
import torch.distributed as dist


def _rewrite_aggs(aggs):
    """Per-rank aggregates: AVG -> SUM of the same expression; one COUNT(*) appended."""
    return [("sum", f) if op == "avg" else (op, f) for op, f in aggs] + [("count", [])]


def _gather_rows(t, group=None):
    """All-gather a (rows, W) int64 tensor with per-rank row counts; returns the concatenation
    in rank order (valid rows only)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(max(sizes), 1)
    pad = torch.zeros((mx, t.shape[1]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def groupby_agg(ctx, cols, key_idx, aggs, preds=(), group=None, local_fn=None, merge_fn=None):
    """Distributed sort-based group-by over row-partitioned columns: local partial
    aggregation, all-gather of the partial groups, exact merge. Every rank returns the
    merged result (same dict layout as Context.groupby_agg)."""
    local_fn = local_fn or ctx.groupby_agg
    merge_fn = merge_fn or ctx.groupby_merge
    raggs = _rewrite_aggs(aggs)
    loc = local_fn(cols, key_idx, raggs, preds)
    G = loc["n_groups"]
    dev = loc["results"][-1].device
    key_dtypes = [cols[k].dtype for k in key_idx]
    pieces = [k.reshape(G, 1).to(torch.int64) for k in loc["keys"]]
    for (op, _), r in zip(raggs, loc["results"]):
        pieces.append(r.reshape(G, 2) if op == "sum" else r.reshape(G, 1).to(torch.int64))
    mat = torch.cat(pieces, dim=1) if pieces else torch.zeros((G, 0), dtype=torch.int64, device=dev)
    allm = _gather_rows(mat.contiguous(), group)
    c = 0
    keys = []
    for dt in key_dtypes:
        keys.append(allm[:, c].to(dt).contiguous())
        c += 1
    partial_by_ragg = []
    for op, _ in raggs:
        if op == "sum":
            partial_by_ragg.append(allm[:, c:c + 2].contiguous())
            c += 2
        else:
            partial_by_ragg.append(allm[:, c].contiguous())
            c += 1
    counts = partial_by_ragg[-1]
    partials = [None if op == "count" else partial_by_ragg[a] for a, (op, _) in enumerate(aggs)]
    return merge_fn(keys, aggs, partials, counts)


def pkfk_join_broadcast(ctx, build_keys, probe_keys, group=None, join_fn=None):
    """Shuffled-layout PK-FK join: all-gather the build side (rank-ordered, so the
    concatenation is the global build table), then join the local probe rows.
    Returns (global build row, local probe row) pairs in probe-row order."""
    join_fn = join_fn or ctx.pkfk_join
    allb = _gather_rows(build_keys.reshape(-1, 1).to(torch.int64), group).reshape(-1)
    return join_fn(allb.to(build_keys.dtype), probe_keys)
