"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration + dram bytes)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, {}
for r in rows:
    if len(r) > 10 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"][:70]
        agg.setdefault(k, {}).setdefault(d["Metric Name"], []).append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    t = v.get("gpu__time_duration.sum", [0])
    rd, wr = v.get("dram__bytes_read.sum", [0]), v.get("dram__bytes_write.sum", [0])
    gbs = (sum(rd) + sum(wr)) / max(sum(t), 1)
    print("%-70s n=%-3d t=%8.3f ms  rd=%6.2f GB wr=%6.2f GB  %6.0f GB/s" % (k, len(t), sum(t) / 1e6, sum(rd) / 1e9, sum(wr) / 1e9, gbs))
