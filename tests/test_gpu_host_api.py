"""The C++ host mirror (paper_2212_05271_b200/host/include/gss/*.hpp) compiled with g++ against the C ABI and
run on the device: the reference's own call sites compile unchanged against these headers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def compile_check(out):
    lib = os.path.join(ROOT, "paper_2212_05271_b200", "lib")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "paper_2212_05271_b200", "host", "include"),
           os.path.join(ROOT, "tests", "host_api_check.cpp"), "-o", out, "-L" + lib, "-lgss_b200",
           "-Wl,-rpath," + lib]
    subprocess.run(cmd, check=True)


def test_host_mirror_compiles(tmp_path):
    from paper_2212_05271_b200 import build
    build.build(verbose=False)
    compile_check(str(tmp_path / "host_api_check"))


@pytest.mark.gpu
def test_host_mirror_runs_on_device(tmp_path):
    exe = str(tmp_path / "host_api_check")
    compile_check(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
