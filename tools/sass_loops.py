"""Loops of a kernel's SASS that hold many DMMA / FFMA2: instruction mix per
loop (LDL / STL inside a mainloop = spills on the hot path).

    python tools/sass_loops.py OBJ_OR_SO REGEX_OF_MANGLED_NAME
"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not re.search(sys.argv[2], name):
        continue
    ins = []
    for l in f.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print("==", subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()[:140])
    for a, t in ins:
        m = re.search(r"BRA[^ ]* .*?(0x[0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a:
            continue
        body = [x for x in ins if tgt <= x[0] <= a]
        nd = sum("DMMA" in x[1] for x in body)
        nf = sum("FFMA2" in x[1] or "F32x2" in x[1] for x in body)
        if nd < 16 and nf < 64:
            continue
        if len(body) > 3000:
            continue
        cnt = lambda k: sum(k in x[1] for x in body)
        print(f"  loop {tgt:#x}-{a:#x} n={len(body)} DMMA={nd} FFMA2={nf} LDS={cnt('LDS')} LDL={cnt('LDL')} "
              f"STL={cnt('STL')} NOP={sum(x[1].startswith('NOP') for x in body)}")
