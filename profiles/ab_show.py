"""Print the A/B bench lines of a tag: python profiles/ab_show.py TAG"""
import glob, json, sys
for f in sorted(glob.glob("gpurun_out/ab_%s_*.json" % sys.argv[1])):
    for l in open(f):
        l = l.strip()
        if l.startswith("{"):
            d = json.loads(l)
            print("%-45s %8.1f  c %8.1f  d %8.1f  frac %.3f/%.3f" % (f.split("/")[-1], d["value"], d.get("compress_gbs", 0),
                  d.get("decompress_gbs", 0), d.get("roofline", {}).get("frac", 0), d.get("roofline", {}).get("other_kernel_frac", 0)))
