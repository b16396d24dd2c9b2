"""Per-kernel register / spill summary of one .cu file (ptxas -v), for checking a change before spending GPU time.

    python tools/ptxas_usage.py paper_2409_20361_b200/csrc/prologue.cu [name-filter]
"""
import os
import re
import subprocess
import sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import nvidia.nccl  # noqa: E402

NI = os.path.join(list(nvidia.nccl.__path__)[0], "include")
src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3", "-lineinfo",
                      "-Xcompiler", "-fPIC", "-I", NI, "-I", os.path.join(R, "include"), "-Xptxas", "-v", "-c", src,
                      "-o", "/tmp/_ptxas_usage.o"], capture_output=True, text=True).stderr
name = None
for line in out.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and name:
        spill = int(m.group(1))
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if flt in name:
            print(f"{int(m.group(1)):4d} regs  spill {spill:5d}  {name}")
        name = None
