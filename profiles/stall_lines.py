"""Top SASS lines by stall samples with the per-reason breakdown.
usage: python stall_lines.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
for d in data:
    for r in reasons:
        tot[r] += int(d[ix[r]] or 0)
T = sum(tot.values())
print("total samples", T, " ".join("%s=%.1f%%" % (r[6:], 100.0 * v / T) for r, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]))
hot = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))[:N]
for i in sorted(hot):
    d = data[i]
    br = sorted(((r[6:], int(d[ix[r]] or 0)) for r in reasons), key=lambda kv: -kv[1])[:3]
    print("%5d %-52s samp=%5s %s" % (i, d[ix["Source"]].strip()[:52], d[ix["Warp Stall Sampling (All Samples)"]],
                                     " ".join("%s:%d" % kv for kv in br if kv[1])))
