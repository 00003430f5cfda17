"""CPU checks of the drop-in boundary: the ctypes mirror agrees with the C header, and the
built library exports every entry point ``include/ptopt_cuda.h`` declares (no compute calls)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2404_18034_b200 import abi, binding

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ptopt_cuda.h"

STRUCTS = {
    "ptopt_vehicle_params": abi.VehicleParams, "ptopt_pipg_config": abi.PipgConfig,
    "ptopt_problem_desc": abi.ProblemDesc, "ptopt_subproblem_shape": abi.SubproblemShape,
    "ptopt_subproblem_arrays": abi.SubproblemArrays, "ptopt_workspace_arrays": abi.WorkspaceArrays,
    "ptopt_dispersion_spec": abi.DispersionSpec, "ptopt_run_record": abi.RunRecord,
}


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ptopt_cuda_[a-z0-9_]+)\s*\(", text)))


def test_struct_sizes_match_the_c_compiler(tmp_path):
    src = tmp_path / "sizes.c"
    lines = ['#include <stdio.h>', '#include "ptopt_cuda.h"', "int main(void) {"]
    for name in STRUCTS:
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
    lines += ['  printf("abi %d\\n", PTOPT_ABI_VERSION);', "  return 0;", "}"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-std=c11", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], check=True, capture_output=True,
                                                 text=True).stdout.splitlines())
    for name, cls in STRUCTS.items():
        assert int(out[name]) == C.sizeof(cls), name
    assert int(out["abi"]) == abi.ABI_VERSION
    assert binding.RECORD_DTYPE.itemsize == C.sizeof(abi.RunRecord)


def test_header_is_plain_c_and_cxx(tmp_path):
    for compiler, std, ext in (("gcc", "-std=c99", "c"), ("g++", "-std=c++17", "cpp")):
        src = tmp_path / f"inc.{ext}"
        src.write_text('#include "ptopt_cuda.h"\nint main(void) { return ptopt_cuda_abi_version() == 0; }\n')
        subprocess.run([compiler, std, "-Wall", "-Werror", "-pedantic", f"-I{ROOT / 'include'}",
                        "-Wno-long-long", "-c", str(src), "-o", str(tmp_path / f"inc_{ext}.o")], check=True)


def test_library_exports_every_declared_entry_point():
    lib = binding.load_library()  # raises when the library has not been built
    declared = declared_functions()
    assert len(declared) >= 20
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing
    assert sorted(binding.EXPORTS) == declared  # the binding's list is the header's list
    assert lib.ptopt_cuda_abi_version() == abi.ABI_VERSION


def test_no_device_means_an_error_not_a_fallback():
    """Without a usable sm_100 device create() must fail loudly (no CPU path)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2404_18034_b200 import scenario

    with pytest.raises(binding.PtoptError) as e:
        binding.Solver(scenario.default_scenario(15).problem_desc())
    assert e.value.code == abi.ERR_CUDA
