"""Median per-kernel time / DRAM bytes from an ncu --csv launch list (tools/prof_ab.sh)."""
import collections, csv, sys
for f in sys.argv[1:]:
    hdr = None
    data = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in csv.reader(open(f)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data[d["Kernel Name"][:60]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    print(f)
    for k, v in data.items():
        t = sorted(v["gpu__time_duration.sum"])
        n = len(t)
        med = lambda key: sorted(v[key])[n // 2] / 1e6 if v.get(key) else float("nan")
        print(f"  {k:60s} n={n:3d} med={t[n // 2] / 1e3:8.2f} us  dram_r={med('dram__bytes_read.sum'):8.2f} MB"
              f"  dram_w={med('dram__bytes_write.sum'):7.2f} MB")
