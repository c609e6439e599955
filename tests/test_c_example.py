"""A plain-C host program builds against include/blocksolve_b200.h and the
library (the non-Python integration path of INTEGRATION.md)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2009_12638_b200", "_lib")


def _build(tmp_path):
    from paper_2009_12638_b200.build import build

    build()
    exe = str(tmp_path / "c_cg_solve")
    cmd = ["gcc", "-O2", "-std=c99", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_cg_solve.c"), "-o", exe, "-L", LIBDIR, "-lbsgpu",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_c_host_builds_and_reports_missing_device(tmp_path):
    exe = _build(tmp_path)
    import torch

    if torch.cuda.is_available():
        pytest.skip("covered by the GPU variant")
    r = subprocess.run([exe, "8"], capture_output=True, text=True)
    assert r.returncode == 2 and "error" in r.stderr


@pytest.mark.gpu
def test_c_host_cg_solve_matches_reference_count(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "64"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("its=231 stop=1")  # config-2 analogue at 64^3
