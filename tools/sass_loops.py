"""Static instruction counts of the loops of one kernel that contain DMMA.

usage: python tools/sass_loops.py <lib.so> <function-name-substring>
Finds backward branches in the cuobjdump SASS of the kernel and, for every loop
whose body holds tensor-core instructions, prints its size and opcode mix --
a CPU-side check of the per-step instruction budget before spending GPU time.
"""
import collections
import re
import subprocess
import sys

lib, name = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
ins, on = [], False
for line in out.splitlines():
    if "Function :" in line:
        on = name in line
        continue
    if not on:
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
print(f"{name}: {len(ins)} instructions")
loops = []
for i, (a, t) in enumerate(ins):
    m = re.search(r"\bBRA(?:\.\w+)*\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr:
            loops.append((addr[tgt], i))
for lo, hi in sorted(set(loops), key=lambda x: x[1] - x[0]):
    body = [t for _, t in ins[lo:hi + 1]]
    nd = sum("DMMA" in t for t in body)
    if nd == 0:
        continue
    ops = collections.Counter()
    for t in body:
        p = t.split()
        op = p[1] if p[0].startswith("@") else p[0]
        ops[op.split(".")[0]] += 1
    print(f"loop {ins[lo][0]:#x}..{ins[hi][0]:#x}: {hi - lo + 1} instructions, {nd} DMMA")
    print("   " + ", ".join(f"{o} {c}" for o, c in ops.most_common(18)))
