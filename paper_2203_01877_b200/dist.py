"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL) for the collectives.

The hot path shards by rows (the paper lists data-parallel execution
as future work). Every rank holds a slice of each column; "global row"
means the position in the rank-ordered concatenation of the ranks' slices, so every
distributed result is compared with -- and equals, bit for bit -- the single-GPU result
over the concatenated table.

  * group-by: local partial aggregation (tqp_groupby_agg, AVG rewritten as SUM + COUNT),
    all-gather of the few partial groups, exact merge (tqp_groupby_merge: int128 sums,
    averages recomputed from merged SUM / COUNT, never averaged);
  * PK-FK join, shuffled layout, two exchanges:
      broadcast build -- the build slices are all-gathered in rank order (the global
      build table), the local probe rows join against it;
      co-partition -- equal-width key ranges from an all-reduced device [min, max]
      (tqp_minmax, tqp_range_splitters: no host round trip), both sides' (key, global
      row) partitioned by key range on the GPU (tqp_partition: histogram, scan, stable
      scatter), one all_to_all per column, the local join gathers the received global
      rows as payload (tqp_pkfk_join_payload) -- pairs come out ascending by global
      probe row because the partition is stable and blocks arrive in rank order;
    a byte cost model (pkfk_cost_bytes) picks the cheaper one;
  * sample sort and the generic SMJ: local libtqp sort,
    splitters from sampled sorted keys, contiguous slices of the sorted columns sent
    with all_to_all, local stable sort / Alg. 1 with createOutput fused
    (tqp_smj_expand_payload). Heavy SMJ keys (a key equal to a splitter spans several
    ranks) are split by output range: the key's left rows are divided among its ranks
    by their ordinal within the key (global: the key's rows on lower ranks + the local
    position), its right rows replicated to each of them.

Collectives go through `_Comm`: NCCL on device tensors; with the gloo backend, device
tensors are staged through host memory (the world-size-2 tests run two ranks on one
GPU that way, and on CPU with the oracle as the local operators). The only host syncs
are the ones a collective's split sizes need (one per exchange) and the tiny splitter
/ heavy-key metadata. The local operators come from `ops` (default: the libtqp context,
so every full-column step runs in libtqp's kernels; the CPU tests pass an oracle-backed
stand-in with the same methods).
"""

import torch
import torch.distributed as dist


# --------------------------------------------------------------------- plumbing

# Exchange instrumentation (bench.py): when a list, every all_to_all_v appends
# (start event, end event, bytes received from other ranks, bytes sent to other ranks).
EXCHANGE_LOG = None


class _Comm:
    """Collectives on one process group; gloo gets host copies of device tensors."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.stage = dist.get_backend(group) == "gloo"

    def _h(self, t):
        return t.cpu() if self.stage and t.is_cuda else t

    def _dev(self):
        """Where small control tensors live: host for gloo, the current GPU for NCCL."""
        return torch.device("cpu") if self.stage else torch.device("cuda", torch.cuda.current_device())

    def all_reduce(self, t, op=dist.ReduceOp.SUM):
        h = self._h(t)
        dist.all_reduce(h, op=op, group=self.group)
        if h is not t:
            t.copy_(h)
        return t

    def barrier(self):
        dist.barrier(group=self.group)

    def all_gather_sizes(self, n):
        """Every rank's element count (one tiny collective + host read)."""
        x = torch.tensor([n], dtype=torch.int64, device=self._dev())
        out = [torch.empty_like(x) for _ in range(self.world)]
        dist.all_gather(out, x, group=self.group)
        return torch.cat(out).tolist()

    def all_gather_cat(self, t, sizes=None):
        """Concatenation of every rank's 1-D tensor in rank order (uneven sizes): one
        broadcast per rank into views of the output (no copy after the collective)."""
        sizes = self.all_gather_sizes(t.numel()) if sizes is None else sizes
        out = torch.empty(sum(sizes), dtype=t.dtype, device=t.device)
        ho = self._h(out) if self.stage else out
        o = 0
        for r, s in enumerate(sizes):
            view = ho[o:o + s]
            if r == self.rank:
                view.copy_(self._h(t))
            if s:
                dist.broadcast(view, src=r, group=self.group)
            o += s
        if ho is not out:
            out.copy_(ho)
        return out

    def exchange_counts(self, counts):
        """counts[d] = rows this rank sends to d (device or host int64, shape (world,) or
        (world, k)) -> (send, recv) host lists; the one host sync of an exchange."""
        hc = counts.to(device=self._dev(), dtype=torch.int64).reshape(self.world, -1).contiguous()
        r = torch.empty_like(hc)
        dist.all_to_all_single(r, hc, group=self.group)
        both = torch.stack([hc, r]).cpu().tolist()
        return both[0], both[1]

    def all_to_all_v(self, t, send, recv):
        """all_to_all_single of a 1-D tensor with host split sizes; blocks arrive in
        source-rank order."""
        out = torch.empty(sum(recv), dtype=t.dtype, device=t.device)
        log = EXCHANGE_LOG is not None and t.is_cuda
        if log:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        if self.stage and t.is_cuda:
            ho = torch.empty(sum(recv), dtype=t.dtype)
            dist.all_to_all_single(ho, t.cpu(), recv, send, group=self.group)
            out.copy_(ho)
        else:
            dist.all_to_all_single(out, t.contiguous(), recv, send, group=self.group)
        if log:
            e1.record()
            es = t.element_size()
            EXCHANGE_LOG.append((e0, e1, (sum(recv) - recv[self.rank]) * es, (sum(send) - send[self.rank]) * es))
        return out


def _offset(comm, n):
    """(global offset of this rank's slice, total rows) from every rank's row count."""
    sizes = comm.all_gather_sizes(n)
    return sum(sizes[:comm.rank]), sum(sizes)


def _key_dtype_ok(t):
    if t.dtype not in (torch.int64, torch.int32, torch.uint8):
        raise TypeError(f"distributed operators take u8 / i32 / i64 key columns, not {t.dtype}")


# ---------------------------------------------------------------------- group-by

def _rewrite_aggs(aggs):
    """Per-rank aggregates: AVG -> SUM of the same expression; one COUNT(*) appended."""
    return [("sum", f) if op == "avg" else (op, f) for op, f in aggs] + [("count", [])]


def groupby_agg(ops, cols, key_idx, aggs, preds=(), group=None, local_fn=None, merge_fn=None):
    """Distributed sort-based group-by over row-partitioned columns: local partial
    aggregation, all-gather of the partial groups, exact merge. Every rank returns the
    merged result (same dict layout as Context.groupby_agg). Aggregates over fp64 value
    columns are rejected: the exact merge is integer (int128) only."""
    for op, factors in aggs:
        if op != "count" and any(cols[c].dtype == torch.float64 for c, _, _ in factors):
            raise ValueError("distributed groupby_agg: fp64 aggregate columns are not supported "
                             "(tqp_groupby_merge merges exact int128 partials only)")
    local_fn = local_fn or ops.groupby_agg
    merge_fn = merge_fn or ops.groupby_merge
    comm = _Comm(group)
    raggs = _rewrite_aggs(aggs)
    loc = local_fn(cols, key_idx, raggs, preds)
    G = loc["n_groups"]
    dev = loc["results"][-1].device
    key_dtypes = [cols[k].dtype for k in key_idx]
    pieces = [k.reshape(G, 1).to(torch.int64) for k in loc["keys"]]
    for (op, _), r in zip(raggs, loc["results"]):
        pieces.append(r.reshape(G, 2) if op == "sum" else r.reshape(G, 1).to(torch.int64))
    mat = torch.cat(pieces, dim=1) if pieces else torch.zeros((G, 0), dtype=torch.int64, device=dev)
    W = mat.shape[1]
    allm = comm.all_gather_cat(mat.contiguous().reshape(-1)).reshape(-1, W)   # a few groups per rank
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


# ------------------------------------------------------------------- PK-FK join

def pkfk_join_broadcast(ops, build_keys, probe_keys, group=None):
    """Shuffled-layout PK-FK join, broadcast build: the build slices all-gathered in rank
    order are the global build table, so left rows come out global; the probe side does
    not move. Returns (global build row, global probe row), ascending probe row."""
    _key_dtype_ok(build_keys)
    comm = _Comm(group)
    poff, _ = _offset(comm, probe_keys.numel())
    allb = comm.all_gather_cat(build_keys)
    lo, ro = ops.pkfk_join(allb, probe_keys)
    if poff:
        ro += poff   # local -> global probe row (the probe side never moved)
    return lo, ro


def pkfk_join_copartition(ops, build_keys, probe_keys, group=None, exchange=None, transport="nccl"):
    """Shuffled-layout PK-FK join by co-partitioning on key ranges (all on the GPU up to the
    all_to_all split sizes). Returns this rank's (global build row, global probe row) pairs
    for its key range, ascending by global probe row; the union over ranks is the
    single-GPU join of the concatenated tables. `exchange` (a dict, optional) receives
    the bytes this rank sent / received."""
    _key_dtype_ok(build_keys)
    _key_dtype_ok(probe_keys)
    comm = _Comm(group)
    G = comm.world
    sizes_b = comm.all_gather_sizes(build_keys.numel())
    sizes_p = comm.all_gather_sizes(probe_keys.numel())
    boff, poff = sum(sizes_b[:comm.rank]), sum(sizes_p[:comm.rank])
    # key ranges: [min, max] of both sides, all-reduced as MIN of (min, ~max) -- ~ reverses order
    mb, mp = ops.minmax(build_keys), ops.minmax(probe_keys)
    lohi = torch.stack([torch.minimum(mb[0], mp[0]), torch.maximum(mb[1], mp[1])])
    red = torch.stack([lohi[0], ~lohi[1]])
    comm.all_reduce(red, op=dist.ReduceOp.MIN)
    lohi = torch.stack([red[0], ~red[1]])
    spl = ops.range_splitters(lohi, G)
    if transport == "p2p":   # the fused partition + exchange over peer memory
        rb_key, rb_row, rp_key, rp_row = _pkfk_exchange_p2p(ops, comm, build_keys, probe_keys, spl, boff, poff,
                                                            exchange)
        (gl,), (gr,), _ = ops.pkfk_join_payload(rb_key, rp_key, [rb_row], [rp_row], indices=False)
        return gl, gr
    bk, brow, bcnt = ops.partition(build_keys, spl, row_base=boff)
    pk, prow, pcnt = ops.partition(probe_keys, spl, row_base=poff)
    send, recv = comm.exchange_counts(torch.stack([bcnt, pcnt], dim=1))
    sb, rb = [s[0] for s in send], [r[0] for r in recv]
    sp, rp = [s[1] for s in send], [r[1] for r in recv]
    rb_key = comm.all_to_all_v(bk, sb, rb)
    rb_row = comm.all_to_all_v(brow, sb, rb)
    rp_key = comm.all_to_all_v(pk, sp, rp)
    rp_row = comm.all_to_all_v(prow, sp, rp)
    if exchange is not None:
        kb_b, kb_p = build_keys.element_size(), probe_keys.element_size()
        me = comm.rank
        exchange["sent_bytes"] = (sum(sb) - sb[me]) * (kb_b + 8) + (sum(sp) - sp[me]) * (kb_p + 8)
        exchange["recv_bytes"] = (sum(rb) - rb[me]) * (kb_b + 8) + (sum(rp) - rp[me]) * (kb_p + 8)
    (gl,), (gr,), _ = ops.pkfk_join_payload(rb_key, rp_key, [rb_row], [rp_row], indices=False)
    return gl, gr


# ------------------------------------------- fused exchange over peer memory (P2P)

class _Arena:
    """This process's receive arena, shared with the other ranks by CUDA IPC (grow-only),
    and the mappings of the other ranks' arenas. With GPUs on NVLink the mappings are P2P
    windows: a partition kernel's stores into them travel over NVLink (the fused
    partition + all-to-all); ranks on one GPU map each other's memory on that GPU."""

    def __init__(self, ops):
        self.ops, self.ptr, self.cap, self.handle, self.gen = ops, None, 0, bytes(64), 0
        self.peers = {}    # rank -> (gen, mapped pointer)

    def sync(self, comm, need):
        """Grow to `need` bytes if necessary, exchange (generation, handle) with every rank,
        (re)map the peers whose arena changed. Returns {rank: base pointer}."""
        old = None
        if need > self.cap:
            old = self.ptr
            self.cap = max(need, 2 * self.cap, 1 << 20)
            self.ptr, self.handle = self.ops.ipc_alloc(self.cap)
            self.gen += 1
        mine = torch.tensor(list(self.gen.to_bytes(8, "little")) + list(self.handle) + [int(old is not None)],
                            dtype=torch.uint8)
        allb = comm.all_gather_cat(mine.to(comm._dev())).cpu().reshape(comm.world, 73)
        bases = {}
        for r in range(comm.world):
            if r == comm.rank:
                bases[r] = self.ptr
                continue
            gen = int.from_bytes(bytes(allb[r, :8].tolist()), "little")
            if r not in self.peers or self.peers[r][0] != gen:
                if r in self.peers:
                    self.ops.ipc_close(self.peers[r][1])
                self.peers[r] = (gen, self.ops.ipc_open(bytes(allb[r, 8:72].tolist())))
            bases[r] = self.peers[r][1]
        if int(allb[:, 72].sum()) > 0:   # some arena moved: once every rank has closed the old
            comm.barrier()               # mappings (above), the owners free the old arenas
            if old is not None:
                self.ops.ipc_free(old)
        return bases


_ARENAS = {}


def _arena(ops):
    key = (id(ops), torch.cuda.current_device())
    if key not in _ARENAS:
        _ARENAS[key] = _Arena(ops)
    return _ARENAS[key]


def _align(x, a=256):
    return (x + a - 1) // a * a


def _pkfk_exchange_p2p(ops, comm, bk, pk, spl, boff, poff, exchange=None):
    """Co-partition exchange by the fused partition: each rank's scatter writes its rows
    straight into the owner ranks' arenas (no send buffer, no NCCL). Returns the received
    (build key, build row, probe key, probe row) as views of this rank's arena, in
    source-rank order like all_to_all."""
    G, me = comm.world, comm.rank
    plan_b, cnt_b = ops.partition_plan(bk, spl)
    plan_p, cnt_p = ops.partition_plan(pk, spl)
    M = comm.all_gather_cat(torch.stack([cnt_b, cnt_p]).reshape(-1).to(comm._dev())).cpu().reshape(G, 2, G).tolist()
    kbs, kps = bk.element_size(), pk.element_size()

    def layout(d):   # byte offsets of rank d's four sections, and its need
        rb = sum(M[s][0][d] for s in range(G))
        rp = sum(M[s][1][d] for s in range(G))
        o_bk = 0
        o_br = _align(o_bk + rb * kbs)
        o_pk = _align(o_br + rb * 8)
        o_pr = _align(o_pk + rp * kps)
        return (o_bk, o_br, o_pk, o_pr), _align(o_pr + rp * 8), rb, rp

    lays = [layout(d) for d in range(G)]
    torch.cuda.synchronize()
    comm.barrier()   # every rank is done reading its arena from the previous exchange
    bases = _arena(ops).sync(comm, lays[me][1])
    log = EXCHANGE_LOG is not None
    if log:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    for side, plan, off, es in ((0, plan_b, boff, kbs), (1, plan_p, poff, kps)):
        kptr, rptr, base = [], [], []
        for d in range(G):
            o = lays[d][0]
            kptr.append(bases[d] + o[2 * side])
            rptr.append(bases[d] + o[2 * side + 1])
            base.append(sum(M[s][side][d] for s in range(me)))   # this source's slot in d's block
        plan.scatter(off, kptr, rptr, base)
    if log:   # the fused partition + transfer kernels (bytes: what crossed to other ranks)
        e1.record()
        EXCHANGE_LOG.append((e0, e1, sum((kbs + 8) * M[s][0][me] + (kps + 8) * M[s][1][me] for s in range(G) if s != me),
                             sum((kbs + 8) * M[me][0][d] + (kps + 8) * M[me][1][d] for d in range(G) if d != me)))
    torch.cuda.synchronize()
    comm.barrier()   # every block has landed in its destination
    plan_b.release()
    plan_p.release()
    (o_bk, o_br, o_pk, o_pr), _, rb, rp = lays[me]
    a = bases[me]
    dev = bk.device
    from paper_2203_01877_b200 import device_view
    if exchange is not None:
        exchange["sent_bytes"] = sum((kbs + 8) * M[me][0][d] + (kps + 8) * M[me][1][d] for d in range(G) if d != me)
        exchange["recv_bytes"] = sum((kbs + 8) * M[s][0][me] + (kps + 8) * M[s][1][me] for s in range(G) if s != me)
        exchange["transport"] = "p2p"
    return (device_view(a + o_bk, rb, bk.dtype, dev), device_view(a + o_br, rb, torch.int64, dev),
            device_view(a + o_pk, rp, pk.dtype, dev), device_view(a + o_pr, rp, torch.int64, dev))


def pkfk_cost_bytes(n_build, n_probe, world, key_bytes=8, row_bytes=8):
    """Bytes received per rank by each shuffled-layout strategy:
    broadcast = every other rank's build keys; co-partition = the (key, row) pairs of
    both sides that belong to another rank's key range (uniform keys)."""
    f = (world - 1) / world
    return {"broadcast": n_build * key_bytes * f,
            "copartition": (n_build + n_probe) / world * (key_bytes + row_bytes) * f}


def pkfk_join_shuffled(ops, build_keys, probe_keys, group=None, strategy="auto", exchange=None, transport="nccl"):
    """Shuffled-layout PK-FK join with the cheaper exchange (or the one asked for).
    Returns (strategy, global build rows, global probe rows); broadcast pairs come in
    local probe order, co-partition pairs by global probe row within the rank's range."""
    comm = _Comm(group)
    if strategy == "auto":
        nb = sum(comm.all_gather_sizes(build_keys.numel()))
        np_ = sum(comm.all_gather_sizes(probe_keys.numel()))
        cost = pkfk_cost_bytes(nb, np_, comm.world)
        strategy = min(cost, key=cost.get)
    if strategy == "broadcast":
        lo, ro = pkfk_join_broadcast(ops, build_keys, probe_keys, group)
        if exchange is not None:
            sizes = comm.all_gather_sizes(build_keys.numel())
            exchange["recv_bytes"] = (sum(sizes) - sizes[comm.rank]) * build_keys.element_size()
            exchange["sent_bytes"] = sizes[comm.rank] * build_keys.element_size() * (comm.world - 1)
        return strategy, lo, ro
    gl, gr = pkfk_join_copartition(ops, build_keys, probe_keys, group, exchange, transport)
    return strategy, gl, gr


# ---------------------------------------------------------- sample sort / SMJ

def _sample_sorted(sk, per_rank):
    """Evenly spaced samples of a sorted column (a few hundred values: plumbing)."""
    n = sk.numel()
    if n == 0:
        return sk.new_empty(0, dtype=torch.int64)
    idx = torch.linspace(0, n - 1, per_rank, device=sk.device).round().to(torch.int64)
    return sk[idx].to(torch.int64)


def _splitters(comm, sorted_keys, per_rank=64):
    """world - 1 splitters at the quantiles of every rank's regular samples."""
    allv = comm.all_gather_cat(_sample_sorted(sorted_keys, per_rank))
    allv = torch.sort(allv)[0]
    if allv.numel() == 0:
        return allv
    pos = torch.tensor([(i * allv.numel()) // comm.world for i in range(1, comm.world)], dtype=torch.int64,
                       device=allv.device)
    return allv[pos]


def _count_sorted(sk, vals):
    """Occurrences of each value in a sorted column, and its first position (binary searches)."""
    skl = sk.to(torch.int64)
    lb = torch.searchsorted(skl, vals, right=False)
    ub = torch.searchsorted(skl, vals, right=True)
    return ub - lb, lb


def _output_splitters(comm, slk, srk, per_rank=256):
    """world - 1 splitters balancing rows + output pairs per rank (the SMJ's work). Keys
    frequent in the samples are candidates; their exact global counts L_k, R_k (binary
    searches in the sorted columns, all-reduced) weigh L_k * R_k pairs beside the rows
    the samples stand for. Splitters sit at the weight quantiles, so a key heavier than a
    rank's share recurs as consecutive splitters and spans several ranks."""
    loc = torch.cat([_sample_sorted(slk, per_rank), _sample_sorted(srk, per_rank)])
    allv = torch.sort(comm.all_gather_cat(loc))[0]
    dev = allv.device
    if allv.numel() == 0:
        return allv
    uk, cnt = torch.unique_consecutive(allv, return_counts=True)
    cand = uk[cnt >= 2]                      # identical on every rank
    nrows = torch.tensor([slk.numel() + srk.numel()], dtype=torch.int64, device=dev)
    comm.all_reduce(nrows)
    counts = torch.stack([_count_sorted(slk, cand)[0], _count_sorted(srk, cand)[0]]).to(dev)
    comm.all_reduce(counts)
    pairs = (counts[0] * counts[1]).to(torch.float64)
    w_sample = float(nrows.item()) / allv.numel()
    keys = torch.cat([allv, cand])
    wts = torch.cat([torch.full((allv.numel(),), w_sample, dtype=torch.float64, device=dev), pairs])
    order = torch.argsort(keys, stable=True)
    keys, cum = keys[order], torch.cumsum(wts[order], 0)
    total = float(cum[-1].item())
    targets = torch.tensor([total * i / comm.world for i in range(1, comm.world)], dtype=torch.float64, device=dev)
    pos = torch.searchsorted(cum, targets).clamp(max=keys.numel() - 1)
    return keys[pos]


def _global_rows(ops, perm, off):
    rows = perm.to(torch.int64)
    return rows + off if off else rows


def sort_samplesort(ops, keys, group=None):
    """Distributed stable sort. Returns this rank's (sorted keys, their global rows); the
    ranks' outputs concatenated in rank order are the stable (key, global row) order of
    the concatenated column."""
    _key_dtype_ok(keys)
    comm = _Comm(group)
    off, _ = _offset(comm, keys.numel())
    sk, perm = ops.sort(keys)
    rows = _global_rows(ops, perm, off)
    spl = _splitters(comm, sk).to(sk.device)
    # dest(k) = #splitters <= k: the sorted column splits into contiguous slices
    b = torch.searchsorted(sk.to(torch.int64), spl, right=True).tolist() if spl.numel() else []
    cuts = [0] + b + [sk.numel()]
    send = [cuts[d + 1] - cuts[d] for d in range(comm.world)]
    send, recv = comm.exchange_counts(torch.tensor(send, dtype=torch.int64))
    send, recv = [s[0] for s in send], [r[0] for r in recv]
    rk = comm.all_to_all_v(sk, send, recv)
    rr = comm.all_to_all_v(rows, send, recv)
    k2, p2 = ops.sort(rk)     # stable: equal keys stay in source-rank, then source order
    return k2, ops.gather(rr, p2)


def smj_join_copartition(ops, left_keys, right_keys, group=None):
    """Distributed generic sort-merge join (Alg. 1) by key-range co-partitioning with
    output-aware splitters and output-range splitting of heavy keys.
    Returns this rank's (global left row, global right row) pairs in (key, left row,
    right row) order; the concatenation over ranks in rank order is the single-GPU join
    of the concatenated columns.

    A key v equal to one or more splitters spans ranks lo..hi (lo = splitters below v,
    hi = splitters up to v). Its L_v left rows are divided among those ranks by ordinal
    within the key -- global ordinal = the key's rows on lower ranks + local position, so
    rank lo + d' takes ordinals [ceil(d' L_v / span), ceil((d'+1) L_v / span)) -- and its
    right rows are replicated to every one of them: each rank emits the key's pairs for
    its left rows, in (l, r) order, and the ranks' outputs stay in global order."""
    _key_dtype_ok(left_keys)
    _key_dtype_ok(right_keys)
    comm = _Comm(group)
    G, me = comm.world, comm.rank
    loff, _ = _offset(comm, left_keys.numel())
    roff, _ = _offset(comm, right_keys.numel())
    slk, pl = ops.sort(left_keys)
    srk, pr = ops.sort(right_keys)
    lrows, rrows = _global_rows(ops, pl, loff), _global_rows(ops, pr, roff)
    spl = _output_splitters(comm, slk, srk).to(slk.device)
    spl_h = spl.tolist()
    nl, nr = slk.numel(), srk.numel()
    if G > 1 and spl.numel():
        # distinct splitter values: local count and first position in the sorted left keys
        vals = torch.unique(spl)
        c_loc, lb = _count_sorted(slk, vals)
        c_all = comm.all_gather_cat(c_loc.to(torch.int64)).reshape(G, -1)          # (rank, value)
        meta = torch.stack([c_loc, lb, c_all[:me].sum(0), c_all.sum(0)]).cpu().tolist()
        info = {}
        for j, v in enumerate(vals.tolist()):
            lo_v = sum(1 for s in spl_h if s < v)
            hi_v = sum(1 for s in spl_h if s <= v)
            info[v] = dict(c=meta[0][j], lb=meta[1][j], base=meta[2][j], L=meta[3][j], lo=lo_v, span=hi_v - lo_v + 1)
        # left: disjoint slices of the sorted column; boundary d splits key v = spl[d - 1]
        cuts = [0]
        for d in range(1, G):
            f = info[spl_h[d - 1]]
            q = -(-((d - f["lo"]) * f["L"]) // f["span"]) - f["base"]   # ceil division
            cuts.append(f["lb"] + min(max(q, 0), f["c"]))
        cuts.append(nl)
        send_l = [cuts[d + 1] - cuts[d] for d in range(G)]
        # right: slices [lb(spl[d - 1]), ub(spl[d])) -- overlapping on heavy keys (replicas)
        srk64 = srk.to(torch.int64)
        lbs = torch.searchsorted(srk64, spl, right=False).tolist()
        ubs = torch.searchsorted(srk64, spl, right=True).tolist()
        rs = [0] + lbs
        re_ = ubs + [nr]
        send_r = [re_[d] - rs[d] for d in range(G)]
        overlap = any(re_[d] > rs[d + 1] for d in range(G - 1))
        if overlap:   # replicated heavy-key runs: materialise the slices back to back
            rk_send = torch.cat([srk[rs[d]:re_[d]] for d in range(G)])
            rr_send = torch.cat([rrows[rs[d]:re_[d]] for d in range(G)])
        else:
            rk_send, rr_send = srk, rrows
    else:
        send_l, send_r = [nl] + [0] * (G - 1), [nr] + [0] * (G - 1)
        rk_send, rr_send = srk, rrows
    send, recv = comm.exchange_counts(torch.tensor([send_l, send_r], dtype=torch.int64).t())
    sl_, rl_ = [s[0] for s in send], [r[0] for r in recv]
    sr_, rr_ = [s[1] for s in send], [r[1] for r in recv]
    rl_key = comm.all_to_all_v(slk, sl_, rl_)
    rl_row = comm.all_to_all_v(lrows, sl_, rl_)
    rr_key = comm.all_to_all_v(rk_send, sr_, rr_)
    rr_row = comm.all_to_all_v(rr_send, sr_, rr_)
    (gl,), (gr,), _ = ops.smj_join_payload(rl_key, rr_key, [rl_row], [rr_row])
    return gl, gr
