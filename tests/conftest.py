import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    # test-harness hook: WINO_TEST_TUNING="key=value,..." applies libwino tuning keys
    # (wino_tuning_set) for a whole pytest process (variant re-runs of test files)
    spec = os.environ.get("WINO_TEST_TUNING", "")
    if spec:
        from paper_1803_10986_b200 import _native
        for item in spec.split(","):
            k, _, v = item.partition("=")
            _native.set_tuning(k.strip(), v.strip())


import pytest  # noqa: E402


@pytest.fixture
def gemm_tuning():
    """Force a contraction tile config for plans created in the test (libwino
    tuning key "gemm"); cleared afterwards."""
    from paper_1803_10986_b200 import _native
    _native.set_tuning("gemm", None)
    yield lambda cfg: _native.set_tuning("gemm", cfg)
    _native.set_tuning("gemm", None)
