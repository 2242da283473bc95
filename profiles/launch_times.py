"""Per-kernel mean duration (us) and DRAM bytes from an ncu --csv launch list."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; k = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); key = (d['ID'], d['Kernel Name'])
        k.setdefault(key, {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
agg = collections.OrderedDict()
for (i, name), m in k.items():
    a = agg.setdefault(name.split('(')[0][:70], [])
    a.append(m)
for name, ms in agg.items():
    t = sum(m.get('gpu__time_duration.sum', 0) for m in ms) / len(ms) / 1000.0
    rd = sum(m.get('dram__bytes_read.sum', 0) for m in ms) / len(ms); wr = sum(m.get('dram__bytes_write.sum', 0) for m in ms) / len(ms)
    print("%-70s n=%3d  %9.1f us  rd %.3f GB  wr %.3f GB" % (name, len(ms), t, rd / 1e9, wr / 1e9))
