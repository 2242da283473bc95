"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of the
dominant kernels, from `ncu --set full` captures (one launch each).
usage: python profiles/make_traffic.py KEY=report.ncu-rep [KEY=report ...]
KEY is "<workload>/<compress|decompress>" as bench.py looks it up."""
import csv, io, json, os, subprocess, sys

out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
try:
    data = json.load(open(out_path))
except Exception:
    data = {}
for arg in sys.argv[1:]:
    key, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    def val(name):
        i = h.index(name)
        x = float(v[i].replace(",", ""))
        unit = u[i]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    data[key] = int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
    print(key, data[key])
json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
