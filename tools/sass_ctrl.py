"""Decode sm_90/sm_100 SASS control words (stall/yield/barriers) from cuobjdump -sass text.
usage: cuobjdump -sass lib.so | python tools/sass_ctrl.py <function-substring> [opcode-filter]"""
import re
import sys
from collections import Counter, defaultdict

fn = sys.argv[1]
opf = sys.argv[2] if len(sys.argv) > 2 else None
lines = sys.stdin.read().splitlines()
inside = False
instrs = []
pending = None
for ln in lines:
    if "Function :" in ln:
        inside = fn in ln
        continue
    if not inside:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", ln)
    if m:
        pending = (m.group(1).strip(), int(m.group(2), 16))
        continue
    m = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", ln)
    if m and pending:
        hi = int(m.group(1), 16)
        word = (hi << 64) | pending[1]
        stall = (word >> 105) & 0xF
        yld = (word >> 109) & 1
        wbar = (word >> 110) & 7
        rbar = (word >> 113) & 7
        wait = (word >> 116) & 0x3F
        op = re.sub(r"^@!?U?P\w+\s+", "", pending[0]).split(" ")[0]
        instrs.append((op, stall, yld, wbar, rbar, wait, pending[0]))
        pending = None
agg = defaultdict(Counter)
for op, st, y, wb, rb, wt, txt in instrs:
    agg[op.split(".")[0]][st] += 1
for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:20]:
    print(f"{op:10s} n={sum(c.values()):4d} stall-hist={dict(sorted(c.items()))}")
if opf:
    for op, st, y, wb, rb, wt, txt in instrs:
        if op.startswith(opf):
            print(st, y, wb, rb, bin(wt), txt)
