import glob
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "paper_2301_04869_b200", "data")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "bipm_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run with -m gpu on a B200)")


def case_path(name: str) -> str:
    return os.path.join(DATA, name + ".m")


def golden_files():
    """reduced-KKT dump fixtures (not the iterates_*.npz solve summaries)"""
    return sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("iterates_"))


@pytest.fixture(scope="session")
def goldens():
    from oracle.fixtures import load_npz
    return {os.path.basename(p)[:-4]: load_npz(p) for p in golden_files()}
