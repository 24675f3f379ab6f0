"""TPC-H-shaped synthetic orders / lineitem columns.

dbgen is not available offline, so the columns follow the TPC-H rules that
matter to the hot path: sparse order keys (8 of every 32), 1..7 lines per order,
fixed-point decimals (scale 1e-2) as int64, dates as int32 days since
1970-01-01, 1-character flags as uint8 ("§4.1 Data
Representation": numeric n x 1 tensors, strings n x m uint8 right-padded).

The generator also records, for every lineitem row, the row of its parent order
(`l_parent`). That array is generator bookkeeping, not join arithmetic; the
PK-FK closed-form pin uses it.
"""

import torch

from .rng import rand_u32, rand_uniform_int

# Day numbers (days since 1970-01-01), SURVEY.md App. C item 4.
DAYS = {
    "1992-01-01": 8035,
    "1994-01-01": 8766,
    "1995-01-01": 9131,
    "1995-03-15": 9204,
    "1995-06-17": 9298,
    "1998-08-02": 10440,
    "1998-09-02": 10471,
}

# stream ids (one per drawn quantity)
_S_ODATE, _S_NLINES, _S_QTY, _S_PART, _S_DISC, _S_TAX, _S_SHIP, _S_RECV, _S_RF, _S_SHUF = range(1, 11)


def orders_count(sf: float) -> int:
    return int(round(1_500_000 * sf))


def orderkey(i):
    """o_orderkey of global orders row i (TPC-H's sparse keys: 8 of every 32 values)."""
    return (i // 8) * 32 + (i % 8) + 1


def spread_orderkeys(l_parent, rank: int, world: int):
    """Shuffled multi-rank layout: re-parent a rank's lineitem slice so
    its rows' orders are spread over every rank's orders slice. Local parent j of rank
    `rank` becomes global orders row j * world + rank (a bijection onto the orders rows of
    all ranks, each rank owning a contiguous range of them). Returns (l_orderkey, global
    parent row)."""
    g = l_parent * world + rank
    return orderkey(g), g


def tpch_orders_lineitem(sf: float, seed: int = 42, device="cpu", layout: str = "shuffled",
                         order_range=None):
    """Generate orders and lineitem for scale factor `sf`.

    order_range=(lo, hi) restricts generation to orders rows [lo, hi) of the full
    table and their lineitems (per-rank partitions, co-partitioned layout); global
    row numbers of lineitem are returned in `l_global_row`.

    Returns (orders: dict, lineitem: dict) of torch tensors on `device`.
    """
    n_o_total = orders_count(sf)
    lo, hi = (0, n_o_total) if order_range is None else order_range
    dev = torch.device(device)
    i = torch.arange(lo, hi, dtype=torch.int64, device=dev)

    o_orderkey = orderkey(i)
    o_orderdate = rand_uniform_int(seed, _S_ODATE, i, DAYS["1992-01-01"], DAYS["1998-08-02"])
    nlines = rand_uniform_int(seed, _S_NLINES, i, 1, 7)

    # global line offset of order `lo` (count of lines of all preceding orders)
    if lo > 0:
        base = 0
        step = 1 << 24
        for a in range(0, lo, step):
            j = torch.arange(a, min(lo, a + step), dtype=torch.int64, device=dev)
            base += int(rand_uniform_int(seed, _S_NLINES, j, 1, 7).sum().item())
    else:
        base = 0

    parent_local = torch.repeat_interleave(torch.arange(hi - lo, dtype=torch.int64, device=dev), nlines)
    n_l = parent_local.numel()
    r = torch.arange(base, base + n_l, dtype=torch.int64, device=dev)  # clustered global line number

    qty = rand_uniform_int(seed, _S_QTY, r, 1, 50)
    n_parts = max(1, int(round(200_000 * sf)))
    partkey = rand_uniform_int(seed, _S_PART, r, 1, n_parts)
    retail = 90000 + ((partkey // 10) % 20001) + 100 * (partkey % 1000)  # cents
    l_extendedprice = qty * retail                                          # cents (qty whole units)
    l_quantity = qty * 100                                                  # scale 1e-2
    l_discount = rand_uniform_int(seed, _S_DISC, r, 0, 10)                  # scale 1e-2
    l_tax = rand_uniform_int(seed, _S_TAX, r, 0, 8)                         # scale 1e-2
    odate = o_orderdate[parent_local]
    l_shipdate = odate + rand_uniform_int(seed, _S_SHIP, r, 1, 121)
    l_receiptdate = l_shipdate + rand_uniform_int(seed, _S_RECV, r, 1, 30)
    coin = rand_uniform_int(seed, _S_RF, r, 0, 1)
    cut = DAYS["1995-06-17"]
    rf = torch.where(l_receiptdate <= cut,
                     torch.where(coin == 0, torch.full_like(coin, ord("R")), torch.full_like(coin, ord("A"))),
                     torch.full_like(coin, ord("N")))
    ls = torch.where(l_shipdate > cut, torch.full_like(coin, ord("O")), torch.full_like(coin, ord("F")))
    l_orderkey = o_orderkey[parent_local]

    lineitem = {
        "l_orderkey": l_orderkey,
        "l_quantity": l_quantity,
        "l_extendedprice": l_extendedprice,
        "l_discount": l_discount,
        "l_tax": l_tax,
        "l_shipdate": l_shipdate.to(torch.int32),
        "l_receiptdate": l_receiptdate.to(torch.int32),
        "l_returnflag": rf.to(torch.uint8),
        "l_linestatus": ls.to(torch.uint8),
        "l_parent": parent_local,          # row of the parent order within this orders slice
        "l_global_row": r,
    }
    if layout == "shuffled":
        # seeded permutation of the row order: argsort of unique 64-bit random keys
        sk = (rand_u32(seed, _S_SHUF, r) << 32) | (r - base)
        order = torch.argsort(sk)
        lineitem = {k: v[order] for k, v in lineitem.items()}
    elif layout != "clustered":
        raise ValueError(f"unknown layout {layout!r}")

    orders = {
        "o_orderkey": o_orderkey,
        "o_orderdate": o_orderdate.to(torch.int32),
        "o_global_row": i,
    }
    return orders, lineitem
