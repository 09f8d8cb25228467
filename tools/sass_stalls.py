"""Static issue-cycle estimate of a SASS address range from the control codes
(stall count bits 105-108 of each 128-bit instruction, yield bit 109).

    python tools/sass_stalls.py OBJ REGEX_OF_MANGLED_NAME START_HEX END_HEX
"""
import re
import subprocess
import sys
from collections import Counter

obj, pat, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3], 16), int(sys.argv[4], 16)
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
on = False
rows = []
cur = None
for l in out.splitlines():
    if "Function :" in l:
        on = re.search(pat, l) is not None
        continue
    if not on:
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l)
    if m:
        cur = [int(m.group(1), 16), m.group(2).strip(), int(m.group(3), 16), None]
        rows.append(cur)
        continue
    m = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", l)
    if m and cur is not None and cur[3] is None:
        cur[3] = int(m.group(1), 16)
tot = Counter()
cnt = Counter()
for a, t, w0, w1 in rows:
    if not (lo <= a <= hi) or w1 is None:
        continue
    ctrl = w1 >> 41  # bits 105.. of the 128-bit word
    stall = ctrl & 0xF
    op = (t.split()[1] if t.startswith("@") else t.split()[0]).split(".")[0]
    tot[op] += max(stall, 1)
    cnt[op] += 1
    if len(sys.argv) > 5:
        print(f"{a:#x} stall={stall:2d} y={(ctrl >> 4) & 1} wb={(ctrl >> 5) & 7} rb={(ctrl >> 8) & 7} wm={(ctrl >> 11) & 63:06b} {t[:70]}")
print("op count issue+stall cycles")
for op, c in tot.most_common():
    print(f"{op:8s} {cnt[op]:5d} {c:6d}")
print("total", sum(cnt.values()), sum(tot.values()))
