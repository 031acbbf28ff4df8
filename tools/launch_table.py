"""Summarise an ncu --csv launch list: per-kernel duration and DRAM bytes."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = d["Metric Value"].replace(",", "")
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
items = list(per.items())[-last:] if last else list(per.items())
for (i, name), m in items:
    short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    print(f"{i:>4} {short:28s} {float(m.get('gpu__time_duration.sum', 0))/1e3:8.2f} us  "
          f"R={float(m.get('dram__bytes_read.sum', 0))/1e6:8.2f} MB W={float(m.get('dram__bytes_write.sum', 0))/1e6:6.2f} MB "
          f"warps={m.get('sm__warps_active.avg.pct_of_peak_sustained_active', '')}")
