import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))
if str(REPO / "tests") not in sys.path:
    sys.path.insert(0, str(REPO / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a CUDA path)")


@pytest.fixture(scope="session")
def built():
    """Native libraries present (builds them in-tree when missing)."""
    from paper_2206_06302_b200 import _build
    lib = REPO / "paper_2206_06302_b200" / "lib"
    need = [lib / "libcoloc_cuda.so", lib / "libcoloc_stream.so", lib / "test_api",
            lib / "test_lambda", lib / "test_launch_policy", lib / "libstream_native.so",
            REPO / "oracle" / "liboracle.so"]
    if not all(p.exists() for p in need):
        _build.build_all()
    return lib
