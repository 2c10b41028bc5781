"""Markdown table of a tools/workloads.py report."""
import json
import sys

d = json.load(open(sys.argv[1]))
print(f"peaks: L2 {d['peaks']['l2_gbs']} GB/s (row staging, live), HBM {d['peaks']['hbm_gbs']} GB/s "
      f"({d['peaks']['hbm_source']})\n")
print("| workload | G | deposit | ants/GPU | construct ms | (kernel) | % L2 roof | update ms | % HBM roof | ms/iter | exchange (modelled) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
ref = {}
for w in d["workloads"]:
    if w.get("impl"):
        ref[(w["workload"], w["deposit"])] = w
        continue
    r = w["roofline"]
    ex = w.get("exchange")
    exs = f"{ex['bytes_per_gpu']/1e6:.0f} MB, {ex['modelled_ms']} ms" if ex else "—"
    print(f"| {w['workload']} | {w['G']} | {w['deposit']} | {w['m_local']} | {w['construct_ms']:.3f} | "
          f"{w['construct_kernel_ms']:.3f} | {100*r['construct']['frac']:.0f}% | {w['update_ms']:.3f} | "
          f"{100*r['update']['frac']:.0f}% | {w['ms_per_iter']:.3f} | {exs} |")
print("\nReference CPU Engine (same run, same host):\n")
print("| workload | deposit | construct ms | update ms | ms/iter | threads |")
print("|---|---|---|---|---|---|")
for (name, dep), w in ref.items():
    print(f"| {name} | {dep} | {w['construct_ms']:.1f} | {w['update_ms']:.1f} | {w['ms_per_iter']:.1f} | {w['cores']} |")
