import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE = "/root/reference/proj"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def _ensure_oracle_libs():
    """Build the checkers if they are missing (only possible where
    /root/reference exists; on the GPU box they arrive prebuilt)."""
    need_ref = not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgbref.so"))
    need_orc = not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so"))
    if need_orc:
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "restatement"], check=True,
                       capture_output=True)
    if need_ref and os.path.isdir(REFERENCE):
        subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True,
                       capture_output=True)


@pytest.fixture(scope="session")
def ref():
    _ensure_oracle_libs()
    from oracle.bindings import Ref

    return Ref()


@pytest.fixture(scope="session")
def orc():
    _ensure_oracle_libs()
    from oracle.bindings import Oracle

    return Oracle()


def golden(scale: int) -> dict:
    with open(os.path.join(GOLDEN, f"rmat_s{scale}.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gbg():
    import paper_2405_11671_b200.graph as g

    return g
