"""The C++ host mirror (include/tpfuse_b200/tpfuse.hpp) through its own C++ test
program (tests/cpp/test_tpfuse_b200.cpp), written like the reference's GTest suites."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_tpfuse_b200")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)


def test_cpp_mirror_schedules_cpu():
    _build()
    r = subprocess.run([BIN, "--cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_mirror_acceptance_gpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, TPF_TIMEOUT_MS="3000"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "Acceptance.C1" in r.stdout and "0 failed" in r.stdout
