import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_CUDA = _has_cuda()


def pytest_collection_modifyitems(config, items):
    if HAS_CUDA:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "rng_golden.json")) as f:
        return json.load(f)


@pytest.fixture(autouse=True)
def _checked_build_guards(request):
    """SMC_CHECKED_RUN=1 with a checked library (SMC_LIB_PATH, built with -DSMC_CHECKED=1;
    tools/gpu/checked.sh): after every GPU test, no kernel index guard may have fired."""
    yield
    if not os.environ.get("SMC_CHECKED_RUN") or "gpu" not in request.keywords or not HAS_CUDA:
        return
    import torch
    from paper_1306_5583_b200 import _abi
    torch.cuda.synchronize()
    checked, fails, where = _abi.check_failures()
    assert checked, "SMC_CHECKED_RUN set but the library is not a checked build"
    assert fails == 0, f"{fails} kernel index guard(s) fired, first at {where}"
