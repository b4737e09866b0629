"""Instruction mix of the innermost loop(s) of a kernel in cuobjdump -sass
output: finds backward branches and counts opcodes between target and branch.

    cuobjdump -sass -fun NAME lib.so | python tools/sass_loop.py
"""
import re
import sys
from collections import Counter

lines = [l for l in sys.stdin.read().splitlines() if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l)]
ins = []
for l in lines:
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, text) in enumerate(ins):
    m = re.search(r"\bBRA\b.*?`?\(?\.L_x_\d+\)?|BRA\s+0x([0-9a-f]+)", text)
    t = re.search(r"BRA(?:\.U)?\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", text)
    if not t or t.group(1) is None:
        continue
    tgt = int(t.group(1), 16)
    if tgt < a and tgt in addr_idx:
        body = ins[addr_idx[tgt]:i + 1]
        ops = Counter()
        for _, tx in body:
            tx = re.sub(r"^@!?U?P\w+\s+", "", tx)
            ops[tx.split()[0]] += 1
        print(f"loop {tgt:#x}-{a:#x}: {len(body)} instructions")
        for op, n in ops.most_common():
            print(f"  {n:4d} {op}")
