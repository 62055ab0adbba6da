"""Register / spill summary of the hot kernels from ptxas -v (build-time check)."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2107_12672_b200/csrc/ddvr_fwd.cu"
extra = sys.argv[2:]
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
       "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-Iinclude", "-Ipaper_2107_12672_b200/csrc", *extra,
       "-c", "-o", "/tmp/regs.o", src]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
fn, spill = None, ""
for line in err.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        fn = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        spill = ""
    # ptxas prints a function's stack / spill line before its register count
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and (m.group(1) != "0" or m.group(2) != "0"):
        spill = f"  [spill st {m.group(1)} ld {m.group(2)}]"
    m = re.search(r"Used (\d+) registers", line)
    if m and fn:
        print(f"{m.group(1):>4} regs  {fn[:100]}{spill}")
