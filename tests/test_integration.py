"""The reference-side binding (integration/gnp_cuda_operator.hpp) compiled
against the REFERENCE's own headers and linked with the unmodified reference
library (oracle/_ref/libgnpref.so) plus libgnpc.so: the reference's
fgmres_solve drives the CUDA GNP operator through its FlexibleOperator
interface (tests/cpp/adapter_check.cpp).  Built by __graft_entry__.build()
where /root/reference exists; the binary travels to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "adapter_check")
REF_INC = "/root/reference/proj/include"


def build_adapter_check():
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", f"-I{REF_INC}", f"-I{ROOT}/include", f"-I{ROOT}/integration",
           os.path.join(ROOT, "tests", "cpp", "adapter_check.cpp"), f"-L{ROOT}/oracle/_ref", "-lgnpref",
           f"-L{ROOT}/paper_2406_00809_b200", "-lgnpc",
           "-Wl,-rpath,$ORIGIN/../../oracle/_ref:$ORIGIN/../../paper_2406_00809_b200", "-o", BIN]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers only in the build container")
def test_adapter_compiles_against_reference_and_flat_order_matches():
    build_adapter_check()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode in (0, 3), r.stdout + r.stderr
    assert "ok flatten" in r.stdout


@pytest.mark.gpu
def test_reference_fgmres_drives_cuda_operator():
    if not os.path.exists(BIN):
        pytest.skip("adapter_check not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok apply vs reference gnn_apply" in r.stdout
    assert "ok iteration parity" in r.stdout
