"""Instruction totals per SASS region (split at lines whose count changes a lot)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
cnt = [int(r[ix["Instructions Executed"]] or 0) for r in data]
smp = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
tot = sum(cnt)
regions = []; start = 0
for i in range(1, len(cnt) + 1):
    if i == len(cnt) or cnt[i] != cnt[start]:
        regions.append((start, i)); start = i
agg = {}
for s, e in regions:
    c = sum(cnt[s:e]); 
    if c: agg[(s, e)] = c
for (s, e), c in sorted(agg.items(), key=lambda kv: -kv[1])[:25]:
    print("lines %5d-%5d  n=%3d  per-line=%10d  total=%11d (%5.1f%%)  samples=%d  first: %s" % (
        s, e - 1, e - s, cnt[s], c, 100.0 * c / tot, sum(smp[s:e]), data[s][ix["Source"]].strip()[:50]))
