"""The C++ mirror of the reference engine (paper_2407_19871_b200/host/locpir_b200.hpp)
compiles against the C ABI (CPU) and passes the reference's own engine/circuit tests
restated in tests/cpp/test_mirror.cpp (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2407_19871_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_mirror")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "test_mirror.cpp"), f"-L{LIBDIR}",
                    "-llocpir_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_cpp_mirror_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_mirror_reference_tests(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
