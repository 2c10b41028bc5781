"""Top stall lines of one kernel in an .ncu-rep (source page, SASS view).
    python tools/ncu_hot.py gpurun_out/x.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ci = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ci[key]] or 0) for r in data) or 1.0
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r in sorted(data, key=lambda r: -float(r[ci[key]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(((float(r[ci[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{float(r[ci[key]]) / tot * 100:5.1f}% {r[ci['Address']][-5:]} {r[ci['Source']].strip()[:58]:58s} "
          + " ".join(f"{s}:{int(v)}" for v, s in top))
