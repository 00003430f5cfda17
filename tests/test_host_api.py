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


def build_example(name="montecarlo_batch"):
    BUILD.mkdir(exist_ok=True)
    exe = BUILD / name
    subprocess.run(
        ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", f"-I{HOST}",
         str(ROOT / "examples" / f"{name}.cpp"), "-o", str(exe), f"-L{LIBDIR}", "-lptopt_cuda",
         f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_example_compiles_and_rejects_bad_input(tmp_path):
    """examples/montecarlo_batch.cpp (config -> run_batch -> CSV): builds, and the argument / config
    errors exit with the reference CLI's usage code before any GPU work."""
    assert subprocess.run([str(build_example("solve_nominal"))], capture_output=True).returncode == 2
    exe = build_example()
    assert subprocess.run([str(exe)], capture_output=True).returncode == 2
    bad = tmp_path / "bad.json"
    bad.write_text('{"vehicle": {"T_min": 9}}')
    out = subprocess.run([str(exe), str(bad)], capture_output=True, text=True)
    assert out.returncode == 2 and "vehicle.T_min must be strictly below vehicle.T_max" in out.stderr


@pytest.mark.gpu
def test_example_batch_from_config_matches_the_binding(tmp_path):
    """The example driven by a JSON configuration writes the runs.csv / summary.csv / trajectory files
    of the same batch that the ctypes harness solves (identical device path, so the CSV numbers
    round-trip to the records bit for bit)."""
    import json

    import numpy as np

    from paper_2404_18034_b200 import scenario
    from paper_2404_18034_b200.binding import Solver

    exe = build_example()
    cfg = {"grid": {"N": 10, "audit_substeps": 8}, "scp": {"max_iters": 3}, "pipg": {"j_max": 200, "power_j_max": 300},
           "montecarlo": {"batch_size": 6, "workers": 2, "converged_floor": 0.0}, "output_dir": str(tmp_path)}
    path = tmp_path / "run.json"
    path.write_text(json.dumps(cfg))
    out = subprocess.run([str(exe), str(path), "--dump-trajectories"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("runs=6 converged_fraction=0.0000")
    rows = [l.split(",") for l in (tmp_path / "runs.csv").read_text().splitlines()[1:]]
    assert len(rows) == 6

    sc = scenario.default_scenario(10)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max, sc.audit_substeps = 3, 200, 300, 8
    spec = sc.dispersion
    with Solver(sc.problem_desc()) as s:
        rec, x, u = s.run_batch(6, 0, sc.initial_state, spec.r_low, spec.r_high, spec.seed, audit_substeps=8,
                                keep_trajectories=True)
    for b, row in enumerate(rows):
        assert int(row[0]) == b and int(row[5]) == rec["scp_iterations"][b] and row[10] == ""
        got = np.array([float(v) for v in row[1:4] + row[6:10]])
        want = np.array([*rec["initial_position"][b], rec["propellant_used"][b], rec["final_defect_inf"][b],
                         rec["max_pointwise_g"][b], rec["max_node_y_increase"][b]])
        assert np.array_equal(got, want), (b, got, want)
    summary = dict(l.split(",") for l in (tmp_path / "summary.csv").read_text().splitlines()[1:])
    assert summary["batch_size"] == "6" and summary["iterations_3"] == "6" and summary["workers"] == "2"
    traj = np.array([[float(v) for v in l.split(",")] for l in (tmp_path / "trajectory_0004.csv").read_text().splitlines()[1:]])
    assert traj.shape == (10, 24)
    assert np.array_equal(traj[:, 2:17], x[4]) and np.array_equal(traj[:, 17:24], u[4])


@pytest.mark.gpu
def test_example_single_solve_from_config_matches_the_binding(tmp_path):
    """examples/solve_nominal.cpp (the reference's `solve` subcommand): config -> initial_guess ->
    scp_solve -> dense audit with samples -> trajectory.csv / dense_audit.csv / diagnostics.txt, against
    the same solve through the ctypes harness (identical device path: bit for bit)."""
    import json

    import numpy as np

    from paper_2404_18034_b200 import scenario
    from paper_2404_18034_b200.binding import Solver

    exe = build_example("solve_nominal")
    cfg = {"grid": {"N": 9, "audit_substeps": 5}, "scp": {"max_iters": 3}, "pipg": {"j_max": 150, "power_j_max": 200},
           "output_dir": str(tmp_path)}
    path = tmp_path / "run.json"
    path.write_text(json.dumps(cfg))
    out = subprocess.run([str(exe), str(path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 1, out.stdout + out.stderr          # three iterations do not converge
    assert out.stdout.startswith("converged=0 iterations=3 ")
    diag = (tmp_path / "diagnostics.txt").read_text().splitlines()
    assert diag[0] == "non-convergence diagnostics" and diag[1] == "iterations 3" and len(diag) == 4 + 3

    sc = scenario.default_scenario(9)
    sc.max_iters, sc.pipg_j_max, sc.power_j_max = 3, 150, 200
    nominal = np.array(sc.initial_state)
    xg, ug = scenario.initial_guess(sc, nominal)
    with Solver(sc.problem_desc()) as s:
        res = s.scp_solve(nominal[None], xg[None], ug[None], np.array([sc.dispersion.seed], np.uint64))
        smp = s.dense_violation_audit_samples(res["x"], res["u"], 5)
    traj = np.array([[float(v) for v in l.split(",")] for l in (tmp_path / "trajectory.csv").read_text().splitlines()[1:]])
    assert np.array_equal(traj[:, 2:17], res["x"][0]) and np.array_equal(traj[:, 17:24], res["u"][0])
    rows = np.array([[float(v) for v in l.split(",")] for l in (tmp_path / "dense_audit.csv").read_text().splitlines()[1:]])
    assert rows.shape == (8 * 6, 12)
    assert np.array_equal(rows, smp["samples"][0].reshape(-1, 12))
