"""JSON run-configuration ingestion: paper_2404_18034_b200/host/ptopt_b200_config.hpp
must read the reference's configuration files (proj/include/ptopt/config.hpp:199-295, 360-370) to
the same RunConfig / problem, and reject what the reference rejects with the same error class and
ConfigError message.

tests/golden/config/expected.txt was written by the reference's own loader (tests/cpp/config_formats.cpp
built with -DWITH_REFERENCE against /root/reference and nlohmann/json 3.11.3, which this container has
under cudnn_frontend's third-party tree; `python tests/test_config_format.py` regenerates it).  The
missing-file case is checked separately (its path is not portable)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HOST = ROOT / "paper_2404_18034_b200" / "host"
BUILD = ROOT / "tests" / "_build"
GOLDEN = ROOT / "tests" / "golden" / "config"
CASES = sorted((GOLDEN / "cases").glob("*.json"))
SRC = ROOT / "tests" / "cpp" / "config_formats.cpp"
REF_INCLUDE = Path("/root/reference/proj/include")
NLOHMANN = Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / "site-packages" / \
    "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"


def run_loader(reference: bool, extra=()):
    BUILD.mkdir(exist_ok=True)
    exe = BUILD / ("config_formats_ref" if reference else "config_formats")
    if reference:
        cmd = ["g++", "-std=c++20", "-O1", "-DWITH_REFERENCE", f"-I{REF_INCLUDE}", f"-I{NLOHMANN}", str(SRC), "-o", str(exe)]
    else:
        cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", f"-I{HOST}", str(SRC),
               "-o", str(exe), f"-L{ROOT / 'paper_2404_18034_b200'}", "-lptopt_cuda",
               f"-Wl,-rpath,{ROOT / 'paper_2404_18034_b200'}"]
    subprocess.run(cmd, check=True)
    return subprocess.run([str(exe), *[str(c) for c in CASES], *extra], check=True, capture_output=True, text=True).stdout


def test_config_loader_matches_the_reference_loader():
    assert len(CASES) == 34
    assert run_loader(False) == (GOLDEN / "expected.txt").read_text()


def test_missing_file_is_a_parse_error(tmp_path):
    out = run_loader(False, extra=[str(tmp_path / "nope.json")])
    assert out.rstrip().endswith("== nope.json\n  ConfigParseError")


def test_golden_expectations_cover_defaults_errors_and_conversions():
    text = (GOLDEN / "expected.txt").read_text()
    blocks = dict(b.split("\n", 1) for b in text.split("== ")[1:])
    assert "grid.N 15\n" in blocks["01_empty_object.json"] and "montecarlo.seed 20260810\n" in blocks["01_empty_object.json"]
    assert "problem.px 1 8 8 8 4 4 4 1 1 1 1 1 1 1 1\n" in blocks["01_empty_object.json"]   # pow2_near of the ranges
    assert "montecarlo.seed 9223372036854775813\n" in blocks["02_full_override.json"]           # > 2^63 survives
    assert "grid.N 50\n" in blocks["04_number_conversions.json"] and "scp.max_iters 1\n" in blocks["04_number_conversions.json"]
    assert "montecarlo.seed 18446744073709551615\n" in blocks["04_number_conversions.json"]     # -1 wraps as in the reference
    assert blocks["05_schema_2.json"] == "  ConfigError: schema: unsupported version 2\n"
    assert blocks["10_tmin_above_tmax.json"] == "  ConfigError: vehicle.T_min must be strictly below vehicle.T_max\n"
    assert blocks["20_trailing_comma.json"] == "  ConfigParseError\n" and blocks["22_empty_file.json"] == "  ConfigParseError\n"
    assert "grid.N 30\n" in blocks["25_duplicate_keys.json"]
    assert blocks["33_bool_for_double.json"] == "  ConfigError: bad value for key 'w_cost'\n"  # a boolean is an int, not a double
    n_err = sum(1 for b in blocks.values() if b.startswith("  Config"))
    assert n_err == 25


@pytest.mark.ref
def test_golden_expectations_are_what_the_reference_loader_gives():
    if not REF_INCLUDE.is_dir() or not (NLOHMANN / "json.hpp").exists():
        pytest.skip("reference tree or nlohmann/json absent")
    assert run_loader(True) == (GOLDEN / "expected.txt").read_text()


if __name__ == "__main__":  # regenerate the expectations from the reference
    (GOLDEN / "expected.txt").write_text(run_loader(True))
    print("wrote", GOLDEN / "expected.txt")
