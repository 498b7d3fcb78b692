"""CPU check of the reference-stream training-pair generator (host side of
gnpc_train_preconditioner's device pairs): tests/cpp/pair_stream_check.cpp
compiled against the product's host sources with the product's flags."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2406_00809_b200", "csrc")


def test_pair_stream_matches_reference_assemble_batch(tmp_path):
    objs = []
    for src, extra in [("host/pair_stream.cpp", ["-O3", "-mavx2"]), ("host/gnp_host.cpp", ["-O2"])]:
        o = str(tmp_path / (os.path.basename(src) + ".o"))
        subprocess.run(["/usr/bin/g++", "-std=c++20", "-fPIC", *extra, "-I", CSRC, "-c",
                        os.path.join(CSRC, src), "-o", o], check=True)
        objs.append(o)
    exe = str(tmp_path / "pair_stream_check")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I", CSRC,
                    os.path.join(ROOT, "tests", "cpp", "pair_stream_check.cpp"), *objs, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok") == 6, r.stdout
