"""The C ABI is usable from plain C without Python: examples/c_api_demo.c
builds against include/casc.h and libcasc.so (CPU), and on a B200 computes a
product with device- and host-resident operands (bitwise the same) close to a
plain double-double dot product (GPU)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    import paper_2303_04353_b200 as casc  # noqa: F401  (the .so exists)
    exe = str(tmp_path / "c_api_demo")
    cmd = ["gcc", "-O2", "-std=c11", "-I" + os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_api_demo.c"),
           "-L" + os.path.join(ROOT, "paper_2303_04353_b200"), "-lcasc",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2303_04353_b200"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_api_demo_builds(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_api_demo_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "320"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_api_demo ok" in r.stdout
