"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL) for the exchanges.

The hot path shards by row ranges (the paper lists data-parallel
execution as future work):
  * group-by: every rank aggregates its rows (tqp_groupby_agg) with AVG rewritten as
    SUM + COUNT; the few partial groups are all-gathered and merged exactly by
    tqp_groupby_merge (int128 sums, averages recomputed from merged SUM / COUNT, never
    averaged);
  * PK-FK join, co-partitioned layout (each rank holds its orders and exactly their
    lineitems): purely local, no exchange;
  * PK-FK join, shuffled layout: either the build side is all-gathered (broadcast
    build) -- the gathered rank-ordered concatenation is the global
    build table, so build rows come out as global row numbers with no remapping -- or
    both sides are co-partitioned by key range (all_to_all of (key, global row)) and
    joined locally; a byte cost model picks the cheaper exchange (pkfk_cost_bytes).
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


def _stable_order(dest, sort_fn):
    """Stable permutation grouping rows by destination rank (libtqp's radix sort on GPUs)."""
    if sort_fn is not None:
        return sort_fn(dest)
    return torch.argsort(dest, stable=True)


def _exchange(cols, dest, world, group=None, sort_fn=None):
    """Send row i of every column to rank dest[i] (all_to_all_single). Received rows are
    in source-rank order, and in source row order within a source."""
    order = _stable_order(dest, sort_fn)
    send_counts = torch.bincount(dest, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    sc, rc = send_counts.tolist(), recv_counts.tolist()
    out = []
    for c in cols:
        r = torch.empty(sum(rc), dtype=c.dtype, device=c.device)
        dist.all_to_all_single(r, c[order].contiguous(), rc, sc, group=group)
        out.append(r)
    return out


def _key_ranges(build_keys, probe_keys, world, group=None):
    """Equal-width key ranges over the global [min, max] of both sides (the TPC-H key
    domain is dense; a sampled splitter set would replace this for skewed keys)."""
    dev = build_keys.device
    big = torch.iinfo(torch.int64)
    lo = torch.tensor([min(int(build_keys.min()) if build_keys.numel() else big.max,
                           int(probe_keys.min()) if probe_keys.numel() else big.max)], dtype=torch.int64, device=dev)
    hi = torch.tensor([max(int(build_keys.max()) if build_keys.numel() else big.min,
                           int(probe_keys.max()) if probe_keys.numel() else big.min)], dtype=torch.int64, device=dev)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    kmin, kmax = int(lo.item()), int(hi.item())
    width = max((kmax - kmin) // world + 1, 1)
    return kmin, width


def pkfk_join_copartition(ctx, build_keys, build_rows, probe_keys, probe_rows, group=None, join_fn=None,
                          sort_fn=None):
    """Shuffled-layout PK-FK join by co-partitioning: both sides' (key, global row) are
    sent to the rank owning the key's range, joined locally, and mapped back to global
    rows. Returns (global build row, global probe row) pairs of this rank's key range,
    ascending by global probe row (the union over ranks = the single-GPU result)."""
    join_fn = join_fn or ctx.pkfk_join
    if sort_fn is None and ctx is not None:
        sort_fn = lambda d: ctx.sort(d)[1]   # noqa: E731
    world = dist.get_world_size(group)
    kmin, width = _key_ranges(build_keys, probe_keys, world, group)
    bk, pk = build_keys.to(torch.int64), probe_keys.to(torch.int64)
    dest_b = torch.clamp((bk - kmin) // width, 0, world - 1)
    dest_p = torch.clamp((pk - kmin) // width, 0, world - 1)
    rb_key, rb_row = _exchange([bk, build_rows.to(torch.int64)], dest_b, world, group, sort_fn)
    rp_key, rp_row = _exchange([pk, probe_rows.to(torch.int64)], dest_p, world, group, sort_fn)
    lo, ro = join_fn(rb_key, rp_key)
    gl, gr = rb_row[lo], rp_row[ro]
    order = _stable_order(gr, sort_fn)
    return gl[order], gr[order]


def pkfk_cost_bytes(n_build, n_probe, world, key_bytes=8, row_bytes=8):
    """Bytes received per rank by each shuffled-layout strategy:
    broadcast = every other rank's build keys; co-partition = the (key, row) pairs of
    both sides that belong to another rank's key range."""
    f = (world - 1) / world
    return {"broadcast": n_build * key_bytes * f,
            "copartition": (n_build + n_probe) / world * (key_bytes + row_bytes) * f}


def pkfk_join_shuffled(ctx, build_keys, build_rows, probe_keys, probe_rows, group=None, strategy="auto",
                       join_fn=None, sort_fn=None):
    """Shuffled-layout PK-FK join with the cheaper exchange (or the one asked for).
    Returns (strategy, global build rows, global probe rows); broadcast pairs come in
    local probe order, co-partition pairs by global probe row within the rank's range."""
    world = dist.get_world_size(group)
    if strategy == "auto":
        n = torch.tensor([build_keys.numel(), probe_keys.numel()], dtype=torch.int64, device=build_keys.device)
        dist.all_reduce(n, group=group)
        cost = pkfk_cost_bytes(int(n[0]), int(n[1]), world)
        strategy = min(cost, key=cost.get)
    if strategy == "broadcast":
        lo, ro = pkfk_join_broadcast(ctx, build_keys, probe_keys, group, join_fn)
        return strategy, lo, probe_rows.to(torch.int64)[ro]
    gl, gr = pkfk_join_copartition(ctx, build_keys, build_rows, probe_keys, probe_rows, group, join_fn, sort_fn)
    return strategy, gl, gr


# ---------------------------------------------------------- distributed sort / SMJ
# SURVEY.md §8(f) NEXT 3. Ranks hold contiguous global row ranges (rank order = global
# row order). Keys are range-partitioned by splitters sampled from every rank's sorted
# keys; (key, global row) pairs are exchanged with all_to_all and sorted / joined locally
# with libtqp. Received blocks arrive in source-rank order, so a stable local sort (or
# the SMJ's (key, left row, right row) order) reproduces the single-GPU order exactly:
# the concatenation of the ranks' outputs, in rank order, is bit-identical to it.

def _splitters(sorted_keys_list, world, group=None, per_rank=64):
    """world - 1 splitters from evenly spaced samples of each rank's keys (exact local
    quantiles when the keys are sorted, a position sample otherwise)."""
    dev = sorted_keys_list[0].device
    samples = []
    for k in sorted_keys_list:
        if k.numel():
            idx = torch.linspace(0, k.numel() - 1, per_rank, device=dev).round().to(torch.int64)
            samples.append(k.to(torch.int64)[idx])
    loc = torch.cat(samples) if samples else torch.empty(0, dtype=torch.int64, device=dev)
    allv = _gather_rows(loc.reshape(-1, 1), group).reshape(-1)
    allv, _ = torch.sort(allv)   # a few thousand host-chosen samples: plumbing, not the operator
    if allv.numel() == 0:
        return torch.empty(0, dtype=torch.int64, device=dev)
    pos = [(i * allv.numel()) // world for i in range(1, world)]
    return allv[torch.tensor(pos, dtype=torch.int64, device=dev)]


def _output_splitters(lk, rk, world, group=None, per_rank=256):
    """world - 1 splitters balancing rows + output pairs per rank (the SMJ's work). Keys
    frequent in a sample are candidates; their exact global counts L_k, R_k are summed
    over the ranks, and each candidate carries its L_k * R_k pairs as weight beside the
    rows the samples stand for. Splitters sit at the weight quantiles, so a key heavier
    than a rank's share recurs as consecutive splitters and spans several ranks."""
    dev = lk.device
    samples = []
    for k in (lk, rk):
        if k.numel():
            sk = torch.sort(k)[0]
            idx = torch.linspace(0, k.numel() - 1, per_rank, device=dev).round().to(torch.int64)
            samples.append(sk[idx])
    loc = torch.cat(samples) if samples else torch.empty(0, dtype=torch.int64, device=dev)
    allv = torch.sort(_gather_rows(loc.reshape(-1, 1), group).reshape(-1))[0]
    if allv.numel() == 0:
        return torch.empty(0, dtype=torch.int64, device=dev)
    uk, cnt = torch.unique_consecutive(allv, return_counts=True)
    cand = uk[cnt >= 2]                      # identical on every rank
    nrows = torch.tensor([lk.numel() + rk.numel()], dtype=torch.int64, device=dev)
    dist.all_reduce(nrows, group=group)
    def count_in(k):   # occurrences of each candidate key in k (candidates are sorted)
        if cand.numel() == 0 or k.numel() == 0:
            return torch.zeros(cand.numel(), dtype=torch.int64, device=dev)
        pos = torch.searchsorted(cand, k)
        hit = cand[pos.clamp(max=cand.numel() - 1)] == k
        return torch.bincount(pos[hit], minlength=cand.numel()).to(torch.int64)
    counts = torch.stack([count_in(lk), count_in(rk)])
    dist.all_reduce(counts, group=group)
    pairs = (counts[0] * counts[1]).to(torch.float64)
    # weighted items: every sample stands for nrows / samples rows; candidates add their pairs
    w_sample = float(nrows.item()) / allv.numel()
    keys = torch.cat([allv, cand])
    wts = torch.cat([torch.full((allv.numel(),), w_sample, dtype=torch.float64, device=dev), pairs])
    order = torch.argsort(keys, stable=True)
    keys, cum = keys[order], torch.cumsum(wts[order], 0)
    total = float(cum[-1].item())
    targets = torch.tensor([total * i / world for i in range(1, world)], dtype=torch.float64, device=dev)
    pos = torch.searchsorted(cum, targets).clamp(max=keys.numel() - 1)
    return keys[pos]


def _range_dest(keys, splitters):
    """Rank owning each key: the number of splitters <= key (equal keys share a rank)."""
    return torch.searchsorted(splitters, keys.to(torch.int64), right=True)


def sort_samplesort(ctx, keys, global_rows, group=None, sort_fn=None):
    """Distributed stable sort. Returns this rank's (sorted keys, their global rows); the
    ranks' outputs concatenated in rank order are the stable (key, global row) order of
    the whole column. sort_fn(k) -> (sorted keys, permutation); default libtqp."""
    sort_fn = sort_fn or ctx.sort
    world = dist.get_world_size(group)
    sk, perm = sort_fn(keys)
    rows = global_rows.to(torch.int64)[perm]
    spl = _splitters([sk], world, group)
    dest = _range_dest(sk, spl)
    rk, rr = _exchange([sk.to(torch.int64), rows], dest, world, group,
                       sort_fn=lambda d: torch.arange(d.numel(), device=d.device))   # sk is sorted: dest ascends
    k2, p2 = sort_fn(rk)
    return k2.to(keys.dtype), rr[p2]


def smj_join_copartition(ctx, left_keys, left_rows, right_keys, right_rows, group=None, join_fn=None,
                         sort_fn=None, n_left_total=None):
    """Distributed generic sort-merge join (Alg. 1) by key-range co-partitioning with
    sampled splitters, with output-range splitting of heavy keys.
    Returns this rank's (global left row, global right row) pairs in (key, left row,
    right row) order; the concatenation over ranks in rank order is the single-GPU result.

    A key equal to one or more splitters is heavy: it spans ranks lo..hi (lo = splitters
    below it, hi = splitters up to it). Its left rows are split across those ranks by
    global left row (row * (hi - lo + 1) // n_left_total: monotone, so each rank gets a
    contiguous range of the key's left rows in order) and its right rows are replicated to
    all of them, so each rank produces the key's pairs for its left rows and the pairs
    still come out in (key, l, r) order across ranks. Light keys go to one rank."""
    join_fn = join_fn or ctx.smj_join
    if sort_fn is None and ctx is not None:
        sort_fn = lambda d: ctx.sort(d)[1]   # noqa: E731
    world = dist.get_world_size(group)
    lk, rk = left_keys.to(torch.int64), right_keys.to(torch.int64)
    lrows, rrows = left_rows.to(torch.int64), right_rows.to(torch.int64)
    if n_left_total is None:   # rows are global offsets into the left column: its length
        t = torch.tensor([lrows.max().item() + 1 if lrows.numel() else 0], dtype=torch.int64, device=lk.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        n_left_total = max(int(t.item()), 1)
    spl = _output_splitters(lk, rk, world, group)
    # left: heavy keys' rows split across their ranks by global row, light rows to one rank
    llo = torch.searchsorted(spl, lk, right=False)
    lhi = torch.searchsorted(spl, lk, right=True)
    dest_l = torch.where(lhi > llo, llo + (lrows * (lhi - llo + 1)) // n_left_total, lhi)
    rl_key, rl_row = _exchange([lk, lrows], dest_l, world, group, sort_fn)
    # right: heavy keys' rows replicated to every rank of the key's span
    rlo = torch.searchsorted(spl, rk, right=False)
    rhi = torch.searchsorted(spl, rk, right=True)
    reps = rhi - rlo + 1
    if bool((reps > 1).any()):
        idx = torch.repeat_interleave(torch.arange(rk.numel(), device=rk.device), reps)
        first = torch.repeat_interleave(torch.cumsum(reps, 0) - reps, reps)
        dest_r = rlo[idx] + (torch.arange(idx.numel(), device=rk.device) - first)
        rk_x, rrows_x = rk[idx], rrows[idx]
    else:
        dest_r, rk_x, rrows_x = rhi, rk, rrows
    rr_key, rr_row = _exchange([rk_x, rrows_x], dest_r, world, group, sort_fn)
    lo, ro = join_fn(rl_key, rr_key)
    return rl_row[lo], rr_row[ro]
