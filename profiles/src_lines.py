"""Per-CUDA-source-line totals of an ncu report (executed warp-instructions and
stall samples), from the correlated cuda+sass source page (needs -lineinfo).
usage: python src_lines.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []; fname = "?"; ix = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No":
        ix = {h: i for i, h in enumerate(r)}; continue
    if ix is None or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        inst = int(r[ix["Instructions Executed"]] or 0); samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    res.append((inst, samp, fname, int(r[0]), r[1].strip()[:70]))
ti = sum(x[0] for x in res) or 1; ts = sum(x[1] for x in res) or 1
print("total warp-instr %d, samples %d" % (ti, ts))
for inst, samp, f, ln, src in sorted(res, key=lambda x: -x[0])[:N]:
    print("%6.2f%% inst %6.2f%% samp  %s:%d  %s" % (100.0 * inst / ti, 100.0 * samp / ts, f, ln, src))
