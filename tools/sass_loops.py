"""List the loops of a kernel's SASS (backward branches) with instruction mix.
usage: python tools/sass_loops.py <obj-or-so> <kernel-substring> [min_hmma]"""
import re
import subprocess
import sys
from collections import Counter

obj, kname = sys.argv[1], sys.argv[2]
min_mma = int(sys.argv[3]) if len(sys.argv) > 3 else 1
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if kname not in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    addr_idx = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, txt) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`?\(?\.L_x_\d+\)?|0x([0-9a-f]+))", txt)
        t = re.search(r"0x([0-9a-f]+)", txt) if "BRA" in txt else None
        if t:
            tgt = int(t.group(1), 16)
            if tgt < a and tgt in addr_idx:
                loops.append((addr_idx[tgt], i))
    print(name, len(ins), "instructions")
    for s, e in sorted(set(loops)):
        body = [x[1].split()[0] if not x[1].startswith("@") else x[1].split()[1] for x in ins[s:e + 1]]
        c = Counter(op.split(".")[0] for op in body)
        if c["HMMA"] < min_mma:
            continue
        print(f"  loop {ins[s][0]:#x}-{ins[e][0]:#x}: {e - s + 1} instr, "
              + ", ".join(f"{k}:{v}" for k, v in c.most_common(14)))
