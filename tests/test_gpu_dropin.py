"""The device containers behind the reference's own C++ harness
(tests/cpp/drop_in.cpp, built by `make -C oracle drop_in` against the
unmodified reference library and libgbg.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "drop_in")


@pytest.mark.gpu
def test_reference_harness_drives_gpu_containers():
    assert os.path.exists(BIN), "oracle/_ref/drop_in not built (run __graft_entry__.build() where /root/reference exists)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
