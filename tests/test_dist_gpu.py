"""Multi-rank dist.py on the CUDA path: two ranks share the one GPU of the test box, the
collectives run over gloo with device tensors staged through host memory (the kernels
never wait on each other), and every local step -- sort, partition, min/max, splitters,
PK-FK join with payload, SMJ with fused createOutput, gather, group-by + merge -- runs in
libtqp. Results are compared element by element with the single-process oracle over the
concatenated slices (tests/_dist_cases.check)."""

import pytest

from _dist_cases import check, run

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(900)
def test_dist_cases_libtqp_two_ranks_one_gpu():
    check(run(2, use_gpu=True), 2)


@pytest.mark.timeout(900)
def test_dist_cases_libtqp_p2p_fused_exchange():
    """The co-partition PK-FK join with the fused exchange: each rank's partition kernel
    writes its rows straight into the owner rank's receive arena through a CUDA IPC
    mapping (on an NVLink node these are peer-GPU stores; here both ranks share the one
    GPU, so the mapping is of the other process's memory on the same device)."""
    check(run(2, use_gpu=True, transport="p2p"), 2)
