"""Pins for the fp64 group-by oracle (oracle.groupby_agg_f64):
a row-by-row Python loop with exact sums (math.fsum) and closed forms."""

import numpy as np

import oracle

# ------------------------------------------------------------ fp64 aggregates

def test_groupby_f64_bruteforce_tiny():
    """The fp64 oracle against a Python loop over rows (grouping by dict, sums by fsum)."""
    import math
    rng = np.random.default_rng(31)
    n = 200
    k = rng.integers(0, 4, n)
    x = rng.normal(0, 1e3, n)
    q = rng.integers(-5, 50, n)
    aggs = [("sum", [(1, 0, 1)]), ("sum", [(1, 0, 1), (2, 100, -1)]), ("min", [(1, 0, 1)]),
            ("max", [(1, 3, -1)]), ("avg", [(1, 0, 1)]), ("count", [])]
    got = oracle.groupby_agg_f64([k, x, q], [0], aggs, [(2, "lt", 40)])
    groups = {}
    for i in range(n):
        if q[i] < 40:
            groups.setdefault(int(k[i]), []).append(i)
    assert [int(v) for v in got["keys"][0]] == sorted(groups)
    for gi, key in enumerate(sorted(groups)):
        rows = groups[key]
        xs = [float(x[i]) for i in rows]
        assert got["results"][0][gi] == math.fsum(xs)
        assert got["results"][1][gi] == math.fsum(float(x[i]) * (100.0 - float(q[i])) for i in rows)
        assert got["results"][2][gi] == min(xs)
        assert got["results"][3][gi] == max(3.0 - v for v in xs)
        assert got["results"][4][gi] == math.fsum(xs) / len(rows)
        assert got["results"][5][gi] == len(rows)


def test_groupby_f64_closed_forms():
    """Constant values: SUM = count * c exactly (c a power of two); no rows -> the empty
    global group (SUM 0, COUNT 0, AVG NaN, MIN +inf, MAX -inf)."""
    n = 1000
    k = np.arange(n) % 7
    c = np.full(n, 0.125)
    got = oracle.groupby_agg_f64([k, c], [0], [("sum", [(1, 0, 1)]), ("count", [])])
    assert got["results"][0] == [0.125 * m for m in got["results"][1]]
    assert sum(got["results"][1]) == n
    e = oracle.groupby_agg_f64([k, c], [], [("sum", [(1, 0, 1)]), ("avg", [(1, 0, 1)]), ("min", [(1, 0, 1)]),
                                            ("max", [(1, 0, 1)]), ("count", [])], [(0, "gt", 100)])
    r = e["results"]
    assert r[0] == [0.0] and np.isnan(r[1][0]) and r[2] == [float("inf")] and r[3] == [float("-inf")] and r[4] == [0]
