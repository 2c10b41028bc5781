"""Top SASS lines by stall samples + key section metrics of an ncu report.
    python tools/ncu_hotspots.py REPORT [kernel-substring] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "Theoretical Occupancy",
        "Eligible Warps Per Scheduler", "L2 Hit Rate", "Executed Instructions")
for r in csv.reader(io.StringIO(det)):
    if len(r) > 14 and ksub in r[4] and r[12] in keep:
        print(f"{r[4][:40]:40s} {r[12]:32s} {r[14]} {r[13]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
                     + (["-k", f"regex:{ksub}"] if ksub else []), capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r)
hdr = rows[hdr_i]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
tot = sum(int(r[iW]) for r in data) or 1
print("total stall samples", tot, "instructions", sum(int(r[iE]) for r in data))
for r in sorted(data, key=lambda r: -int(r[iW]))[:N]:
    print(f"{100*int(r[iW])/tot:5.1f}% exec={int(r[iE]):>10d} {r[iS].strip()[:80]}")
agg = {}
for r in data:
    for i, x in enumerate(hdr):
        if x.startswith("stall_") and "Not Issued" not in x:
            agg[x[6:]] = agg.get(x[6:], 0.0) + float(r[i] or 0)
print("stall reasons (% of samples):",
      ", ".join(f"{k} {100 * v / tot:.1f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
