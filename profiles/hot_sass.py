"""Summarise an ncu source page (SASS view): top instructions by executed
warp-instructions and by stall samples.  usage: python hot_sass.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
tot_inst = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
tot_samp = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total warp-instr %d, stall samples %d, sass lines %d" % (tot_inst, tot_samp, len(data)))
# group by address order, print windows of hot code
hot = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Instructions Executed"]] or 0))[:N]
for i in sorted(hot):
    r = data[i]
    print("%5d %-60s inst=%10s samp=%6s" % (i, r[ix["Source"]].strip()[:60], r[ix["Instructions Executed"]],
                                          r[ix["Warp Stall Sampling (All Samples)"]]))
