"""Multi-rank tests (CPU, gloo) of the exchange logic in paper_2203_01877_b200/dist.py:
key-range partitioning, all_to_all split sizes, broadcast build, heavy-key output-range
splitting, distributed group-by merge. The local operators are oracle-backed stand-ins
(tests/_dist_cases.OracleOps); the expected results are the single-process oracle over
the rank-ordered concatenation of the slices. tests/test_dist_gpu.py runs the same cases
with libtqp's kernels on a GPU."""

import pytest

from _dist_cases import check, run


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_dist_cases_oracle_ops(world):
    check(run(world, use_gpu=False), world)
