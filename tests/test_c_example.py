"""The C ABI from plain C (examples/solve_panda.c): compiles against
include/hjcd.h + libhjcd.so with gcc (CPU), and on a B200 solves 256 Panda
targets through hjcd_solve_host with host buffers (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2510_07514_b200")


def _build(tmp_path):
    exe = str(tmp_path / "solve_panda")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "solve_panda.c"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + LIBDIR, "-lhjcd",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-Wl,-rpath," + LIBDIR, "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles(hjcd_lib, tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_example_solves(hjcd_lib, cuda, tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "256"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    parts = out.stdout.split()
    assert parts[0] == "targets" and int(parts[3]) == 256, out.stdout
    assert float(parts[5]) < 1e-3
