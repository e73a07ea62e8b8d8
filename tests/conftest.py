import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _gpu_available() -> bool:
    try:
        from paper_2110_12952_b200 import _abi
        return _abi.lib().nbbgpu_device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # gpu tests are selected explicitly with -m gpu; without a GPU they fail loudly
    # (no silent skips on the GPU box), but on a CPU-only box they are skipped.
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords and not os.environ.get("NBB_REQUIRE_GPU"):
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    import oracle
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        oracle.build()
    from paper_2110_12952_b200 import build
    build.build()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_long():
    path = os.path.join(GOLDEN, "golden_long.json")
    if not os.path.exists(path):
        return {}
    with open(path) as fh:
        return json.load(fh)


def desc_from_trace(t):
    from paper_2110_12952_b200.descriptor import FractalDescriptor
    return FractalDescriptor(t["fractal"].lstrip("@"), t["k"], t["s"],
                             [tuple(p) for p in t["replicas"]])
