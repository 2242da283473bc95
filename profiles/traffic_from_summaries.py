"""Update profiles/ncu_traffic.json from ncu_summary.py text summaries
(dram__bytes_read.sum + dram__bytes_write.sum of the one captured launch).
usage: python profiles/traffic_from_summaries.py KEY=summary.txt [...]
KEY is "<workload>/<compress|decompress>" as bench.py looks it up."""
import json, os, re, sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
for arg in sys.argv[1:]:
    key, path = arg.split("=", 1)
    tot = 0.0
    for line in open(path):
        m = re.match(r"\s*dram__bytes_(read|write)\.sum\s+([\d.]+)\s+(\w+)", line)
        if m:
            tot += float(m.group(2)) * UNIT[m.group(3)]
    data[key] = int(tot)
    print(key, data[key])
json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
