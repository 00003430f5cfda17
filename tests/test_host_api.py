"""The C++ host mirror of the reference solver API (paper_2404_18034_b200/host/ptopt_b200.hpp).

CPU: it compiles and links against the C-ABI library; with /root/reference present it also
compiles against the reference's own types (drop-in check).  GPU: tests/cpp/test_host_api.cpp
runs every mirrored entry point against the CPU oracle."""
import subprocess
from pathlib import Path

import pytest

from oracle_lib import build_oracle

ROOT = Path(__file__).resolve().parent.parent
HOST = ROOT / "paper_2404_18034_b200" / "host"
LIBDIR = ROOT / "paper_2404_18034_b200"
ORACLE = ROOT / "oracle"
BUILD = ROOT / "tests" / "_build"
REF_INCLUDE = Path("/root/reference/proj/include")


def build_host_test():
    build_oracle()
    BUILD.mkdir(exist_ok=True)
    exe = BUILD / "test_host_api"
    subprocess.run(
        ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", f"-I{HOST}",
         f"-I{ORACLE}", str(ROOT / "tests" / "cpp" / "test_host_api.cpp"), "-o", str(exe),
         f"-L{LIBDIR}", f"-L{ORACLE / '_build'}", "-lptopt_cuda", "-lptopt_oracle",
         f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{ORACLE / '_build'}"], check=True)
    return exe


def test_host_mirror_compiles_and_links():
    assert build_host_test().exists()


@pytest.mark.ref
def test_host_mirror_accepts_the_reference_types():
    if not REF_INCLUDE.is_dir():
        pytest.skip("reference tree absent")
    subprocess.run(
        ["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}", f"-I{HOST}", f"-I{REF_INCLUDE}",
         str(ROOT / "tests" / "cpp" / "compile_with_reference.cpp")], check=True)


@pytest.mark.gpu
def test_host_mirror_against_oracle_on_gpu():
    exe = build_host_test()
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all host-API checks passed" in out.stdout
