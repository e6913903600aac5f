"""The C ABI from plain C (tests/c_abi/spmm_smoke.c): compiled with gcc
against include/svdrec_b200.h and linked to libsvdrec_b200.so -- no Python
or torch between the caller and the library."""
from __future__ import annotations

import shutil
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_consumer_spmm(gpu, tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib = ROOT / "paper_2009_02251_b200"
    exe = tmp_path / "spmm_smoke"
    subprocess.run([cc, "-O2", "-std=c11", str(ROOT / "tests" / "c_abi" / "spmm_smoke.c"), "-I", str(ROOT / "include"),
                    "-I", "/usr/local/cuda/include", "-L", str(lib), "-lsvdrec_b200", "-L", "/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(out.stdout, out.stderr)
    assert out.returncode == 0 and "PASS" in out.stdout
