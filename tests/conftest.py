import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU or GPU runs")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the library / oracle if missing or stale (no-op when up to date)."""
    from paper_1807_00672_b200 import build
    build.build_library()
    build.build_oracle()
    build.build_api_driver()


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def coracle():
    from oracle.pyoracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def refo():
    from oracle.pyoracle import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref (the compiled reference) is not available")
    return RefOracle()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def bit_equal(a, b):
    return np.array_equal(bits(a), bits(b))


def random_state(n, seed, dry_frac=0.0):
    """test_engine.cpp:40-52 (h ~ U(0.2,2), u ~ U(-1,1)) + optional dry mix
    (test_kernels.cpp:185-201)."""
    rng = np.random.default_rng(seed)
    h = rng.uniform(0.2, 2.0, n)
    if dry_frac:
        h[rng.random(n) < dry_frac] = 0.0
    qx = h * rng.uniform(-1, 1, n)
    qy = h * rng.uniform(-1, 1, n)
    return h, qx, qy
