"""Registers / stack / spills of every kernel from the build's ptxas -v logs (build/csrc/*.ptxas.log):
python tools/ptxas_summary.py > profiles/r01_s4_ptxas.txt"""
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
logs = sorted((ROOT / "build" / "csrc").glob("*.ptxas.log"))
if not logs:
    sys.exit("no ptxas logs: run `make -C paper_2404_18034_b200/csrc` first")
print("# ptxas -v summary of every kernel (nvcc 12.9, -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo)")
for log in logs:
    text = log.read_text()
    for m in re.finditer(r"Compiling entry function '(\S+)' for 'sm_100a'\n.*?\n\s*(\d+) bytes stack frame, (\d+) bytes spill stores, "
                         r"(\d+) bytes spill loads\nptxas info\s*: Used (\d+) registers, (.*)", text):
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"ptopt_b200::(\(anonymous namespace\)::|<unnamed>::)?", "", name)
        name = re.sub(r"\(.*$", "", name)
        print(f"{log.stem.replace('.ptxas', ''):16s} {name:44s} regs {int(m.group(5)):3d}  stack {int(m.group(2)):4d} B  "
              f"spill st/ld {m.group(3)}/{m.group(4)} B  {m.group(6)}")
