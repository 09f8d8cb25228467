O=gpurun_out/r02h
mkdir -p $O
MDGEMM_DUAL_LOG=$O/dual_full.log timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-serial > $O/bench_log.json 2> $O/bench_log.err; echo rc=$?
python - <<'PY'
import re
L = open("gpurun_out/r02h/dual_full.log").read().splitlines()
rows = [l for l in L if "launch" in l and "measured" in l]
# keep the last batch (the timed/extra step)
print(len(rows), "launch lines")
tot = dict(ms=0, dcrit=0, fcrit=0, dlate=0.0, flate=0.0)
for l in rows[-115:]:
    m = re.search(r"D\s+(\d+) est\s+([\d.]+) end\s+([\d.]+) \| F\s+(\d+) est\s+([\d.]+) end\s+([\d.]+) \| measured\s+([\d.]+) ms \| ([\d.]+) \+ ([\d.]+)", l)
    if not m: continue
    dend, fend, ms = float(m.group(3)), float(m.group(6)), float(m.group(7))
    tot["ms"] += ms
    if dend >= fend: tot["dcrit"] += 1; tot["dlate"] += dend - fend
    else: tot["fcrit"] += 1; tot["flate"] += fend - dend
print(tot)
PY
tail -40 $O/dual_full.log
