"""TPC-H Q1 / Q6 shapes as neutral descriptors (column lists, predicates, aggregates).

A descriptor is data, not arithmetic: both the oracle and the CUDA binding
interpret it. Predicates are (col, op, value); an aggregate is
(op, [(col, add, sign), ...]) meaning op over prod_f (add_f + sign_f * col_f)
in int64 fixed point (reading R16: decimals scale 1e-2; PAPER.md:1103-1110
"§5.1 Expressions": e.g. sum(l_extendedprice * (1 - l_discount))).
"""

from .tpch import DAYS

Q1_COLS = ["l_returnflag", "l_linestatus", "l_quantity", "l_extendedprice", "l_discount", "l_tax", "l_shipdate"]
Q1_KEYS = [0, 1]
Q1_PREDS = [(6, "le", DAYS["1998-09-02"])]
Q1_AGGS = [
    ("sum", [(2, 0, 1)]),                                  # sum_qty            (scale 1e-2)
    ("sum", [(3, 0, 1)]),                                  # sum_base_price     (1e-2)
    ("sum", [(3, 0, 1), (4, 100, -1)]),                    # sum_disc_price     (1e-4)
    ("sum", [(3, 0, 1), (4, 100, -1), (5, 100, 1)]),       # sum_charge         (1e-6)
    ("avg", [(2, 0, 1)]),                                  # avg_qty
    ("avg", [(3, 0, 1)]),                                  # avg_price
    ("avg", [(4, 0, 1)]),                                  # avg_disc
    ("count", []),                                         # count_order
]
Q1_AGG_NAMES = ["sum_qty", "sum_base_price", "sum_disc_price", "sum_charge",
                "avg_qty", "avg_price", "avg_disc", "count_order"]

Q6_COLS = ["l_shipdate", "l_discount", "l_quantity", "l_extendedprice"]
Q6_PREDS = [(0, "ge", DAYS["1994-01-01"]), (0, "lt", DAYS["1995-01-01"]),
            (1, "ge", 5), (1, "le", 7), (2, "lt", 2400)]
Q6_AGGS = [("sum", [(3, 0, 1), (1, 0, 1)])]               # revenue = sum(price * disc) (1e-4)


def columns(table: dict, names):
    return [table[c] for c in names]
