"""Per-kernel mean duration / DRAM bytes from an ncu --csv launch list."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        try:
            agg[r[iK].split("(")[0][-40:]][r[iM]].append(float(r[iV].replace(",", "")))
        except ValueError:
            pass
    print(path)
    for k, d in agg.items():
        t = d.get("gpu__time_duration.sum", [0])
        rd, wr = d.get("dram__bytes_read.sum", [0]), d.get("dram__bytes_write.sum", [0])
        unit = 1e-3  # ncu reports ns? normalise below
        print(f"  {k:42s} n={len(t):3d} mean={sum(t)/len(t):10.1f} last={t[-1]:10.1f}  "
              f"dram_rd={sum(rd)/len(rd)/1e6:8.1f}MB dram_wr={sum(wr)/len(wr)/1e6:8.1f}MB")
