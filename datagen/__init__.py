"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no sort, join, histogram, group-by
or filter logic). It only draws TPC-H-shaped and Zipf-distributed columns from a
counter-based hash so that any row range can be generated independently on CPU
or GPU with identical integer values (the paper itself only
cites dbgen, "§6 Experimental setup").

Everything is plain torch integer arithmetic, so the same code runs on a CPU
tensor (oracle tests) or a CUDA tensor (bench, full-size parity tests).
"""

from .rng import rand_u32, rand_uniform_int, rand_unit_f64
from .tpch import tpch_orders_lineitem, DAYS
from .keys import zipf_ranks, zipf_keys, uniform_keys, random_small_keys

__all__ = [
    "rand_u32", "rand_uniform_int", "rand_unit_f64",
    "tpch_orders_lineitem", "DAYS",
    "zipf_ranks", "zipf_keys", "uniform_keys", "random_small_keys",
]
