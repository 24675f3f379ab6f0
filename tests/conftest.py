import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtqp.so")
    config.addinivalue_line("markers", "slow: large-size checks")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def sf001():
    """TPC-H-shaped SF0.01 (15K orders, ~60K lineitem), shuffled, seed 42 (BASELINE.json configs[0])."""
    from datagen import tpch_orders_lineitem
    return tpch_orders_lineitem(0.01, seed=42, device="cpu", layout="shuffled")


Q1_SHIPDATE_MAX = 10471  # 1998-09-02 (TPC-H Q1: l_shipdate <= date '1998-12-01' - 90 days)


@pytest.fixture(autouse=True)
def _checked_mode_guards(request):
    """Checked mode (TQP_ALLOC_EXACT=1, tools/gpu_checked.sh): after every GPU test, no
    canary after a libtqp temporary may have been overwritten."""
    yield
    if os.environ.get("TQP_ALLOC_EXACT") == "1" and request.node.get_closest_marker("gpu"):
        import paper_2203_01877_b200 as T
        assert T.context().guard_violations() == 0, "libtqp wrote past the end of a temporary"
