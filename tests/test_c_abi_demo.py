"""The C ABI used from plain C (examples/c_abi_demo.c): it compiles and links against
libmfp.so with gcc (CPU), and on a B200 it solves x^2 - y^2 to 1e-5 (GPU)."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

LIBDIR = os.path.join(ROOT, "paper_2308_14258_b200")


def build(out):
    cmd = ["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", LIBDIR, "-l:libmfp.so", "-L/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_demo_builds(tmp_path):
    build(str(tmp_path / "mfp_demo"))


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = str(tmp_path / "mfp_demo")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "converged 1" in r.stdout
