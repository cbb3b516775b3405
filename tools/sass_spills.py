"""List the backward-branch loops of a kernel's SASS that contain HMMA/UTCHMMA
and the local-memory (spill) instructions inside them.

    cuobjdump -sass -fun <mangled> build/obj/gemv.cu.o > k.sass
    python tools/sass_spills.py k.sass
"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, t) in enumerate(ins):
    m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr_idx:
            loops.append((addr_idx[tgt], i))
for s, e in loops:
    body = [t for _, t in ins[s:e + 1]]
    mma = sum("HMMA" in t or "UTCHMMA" in t for t in body)
    spill = [t for t in body if re.search(r"\b(LDL|STL)\b", t)]
    if mma:
        print(f"loop 0x{ins[s][0]:x}-0x{ins[e][0]:x}: {e - s + 1} instr, {mma} mma, {len(spill)} local")
