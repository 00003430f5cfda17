"""Output formats either side of the hot path: mc::aggregate, node_times and the
runs / summary / trajectory CSV writers of paper_2404_18034_b200/host/ptopt_b200_io.hpp must be
byte-identical to the reference's csv.hpp / montecarlo.hpp.

tests/golden/io/*.csv were written by the reference's own writers (tests/cpp/io_formats.cpp built
with -DWITH_REFERENCE against /root/reference; `python tests/test_io_formats.py` regenerates
them).  The pin is re-checked whenever the reference tree is present."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HOST = ROOT / "paper_2404_18034_b200" / "host"
BUILD = ROOT / "tests" / "_build"
GOLDEN = ROOT / "tests" / "golden" / "io"
REF_INCLUDE = Path("/root/reference/proj/include")
SRC = ROOT / "tests" / "cpp" / "io_formats.cpp"
FILES = ("runs.csv", "summary.csv", "summary_none.csv", "trajectory.csv", "dense_audit.csv", "dense_audit_empty.csv")


def run_writer(reference: bool, out_dir: Path):
    BUILD.mkdir(exist_ok=True)
    out_dir.mkdir(parents=True, exist_ok=True)
    exe = BUILD / ("io_formats_ref" if reference else "io_formats")
    if reference:
        cmd = ["g++", "-std=c++20", "-O1", "-DWITH_REFERENCE", f"-I{REF_INCLUDE}", str(SRC), "-o", str(exe)]
    else:
        cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", f"-I{HOST}",
               str(SRC), "-o", str(exe), f"-L{ROOT / 'paper_2404_18034_b200'}", "-lptopt_cuda",
               f"-Wl,-rpath,{ROOT / 'paper_2404_18034_b200'}"]
    subprocess.run(cmd, check=True)
    subprocess.run([str(exe), str(out_dir)], check=True)


def test_csv_writers_match_the_reference_bytes(tmp_path):
    run_writer(False, tmp_path)
    for name in FILES:
        assert (tmp_path / name).read_bytes() == (GOLDEN / name).read_bytes(), name


def test_golden_csv_files_cover_the_edge_cases():
    runs = (GOLDEN / "runs.csv").read_text().splitlines()
    assert runs[0].endswith("failure,wall_time") and len(runs) == 13
    assert "propagation diverged; interval 3;second line; with commas" in runs[5]  # sanitised failure text
    assert ",-0," in runs[3]                                                      # signed zero survives
    assert "4.9406564584124654e-324" in runs[8]                                   # denormal round trip
    none = dict(l.split(",") for l in (GOLDEN / "summary_none.csv").read_text().splitlines()[1:])
    assert none["converged_fraction"] == "0" and none["propellant_mean"] == "0" and none["iterations_30"] == "1"


@pytest.mark.ref
def test_golden_csv_files_are_what_the_reference_writes(tmp_path):
    if not REF_INCLUDE.is_dir():
        pytest.skip("reference tree absent")
    run_writer(True, tmp_path)
    for name in FILES:
        assert (tmp_path / name).read_bytes() == (GOLDEN / name).read_bytes(), name


if __name__ == "__main__":  # regenerate the fixtures from the reference
    run_writer(True, GOLDEN)
    print("wrote", [str(GOLDEN / f) for f in FILES])
