"""List the loops (backward branches) of one kernel's SASS with their instruction mix.

usage: python tools/sass_loops.py <object.o> <mangled-substring> [min_len]
"""
import re
import subprocess
import sys
from collections import Counter

obj, key = sys.argv[1], sys.argv[2]
min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 20
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs if f.split("\n", 1)[0].strip().endswith(key) or key in f.split("\n", 1)[0])
ins = []
for line in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, text) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*|)0x([0-9a-f]+)", text) or re.search(r"BRA .*?0x([0-9a-f]+)", text)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr_idx:
        continue
    j = addr_idx[tgt]
    n = i - j + 1
    if n < min_len:
        continue
    ops = Counter()
    for _, t in ins[j:i + 1]:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        ops[op.split(".")[0]] += 1
    keys = ("LDL", "STL", "LDG", "LDS", "MUFU", "RED", "REDG", "FFMA", "FFMA2", "FMUL", "FMUL2", "FADD", "FADD2", "IMAD", "IADD3", "I2F", "F2I", "FRND", "DADD", "F2F", "SHF", "LOP3", "ISETP", "FSETP", "SEL", "FSEL", "FMNMX", "BRA")
    print(f"loop 0x{tgt:05x}-0x{a:05x}: {n:4d} instr  " + " ".join(f"{k}={ops[k]}" for k in keys if ops[k]))
