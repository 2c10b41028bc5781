"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py --full gpurun_out/prof.ncu-rep \
        --launches gpurun_out/launches.csv --tag r01

Writes profiles/ncu_summary.json (read by bench.py for roofline.traffic) and
profiles/ncu_<tag>_{full,launches}.txt.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_red.sum",
        "lts__t_sectors_op_atom.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.max"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        res.append({"kernel": d.get("Kernel Name", ""),
                    **{k: d.get(k) for k in KEYS if k in d},
                    "units": {k: u for k, u in zip(hdr, units) if k in KEYS}})
    return res


def to_bytes(v, unit):
    x = float(str(v).replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}.get(unit, 1)
    return x * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = {}
    if os.path.exists(summary_path):
        summary = json.load(open(summary_path))
    if a.full:
        rows = raw(a.full)
        with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}_full.json"), "w") as f:
            json.dump(rows, f, indent=1)
        for r in rows:
            if "construct_roulette" in r["kernel"]:
                u = r["units"]
                dr = to_bytes(r["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
                dw = to_bytes(r["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
                lts = float(str(r["lts__t_sectors.sum"]).replace(",", "")) * 32
                summary.update({"tag": a.tag, "construct_kernel": r["kernel"],
                                "construct_dram_bytes_per_launch": int(dr + dw),
                                "construct_lts_bytes_per_launch": int(lts),
                                "construct_ncu_duration": r["gpu__time_duration.sum"],
                                "construct_ncu_duration_unit": u["gpu__time_duration.sum"],
                                "construct_lts_throughput_pct":
                                    r.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                                "construct_sm_throughput_pct":
                                    r.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                                "construct_registers": r.get("launch__registers_per_thread")})
                break
    if a.launches:
        text = open(a.launches).read()
        lines = [l for l in text.splitlines() if l.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr = rows[0]
        ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        per = collections.defaultdict(list)
        for r in rows[1:]:
            # bench.py's roofline probes and its L2-flush fill are not part of the step
            if "<unnamed>::k_" in r[ik] or "FillFunctor" in r[ik]:
                continue
            v = float(r[iv].replace(",", ""))
            v = v / 1e3 if r[iu] in ("ns", "nsecond") else (v * 1e3 if r[iu] in ("ms", "msecond") else v)
            per[r[ik].split("(")[0]].append(v)  # usecond
        tot = sum(sum(v) for v in per.values())
        share = {k: {"launches": len(v), "total_us": round(sum(v), 1),
                     "share": round(sum(v) / tot, 4)} for k, v in per.items()}
        summary["launch_shares_" + a.tag] = dict(sorted(share.items(),
                                                        key=lambda kv: -kv[1]["total_us"]))
        with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}_launches.txt"), "w") as f:
            for k, v in summary["launch_shares_" + a.tag].items():
                f.write(f"{v['share']*100:6.2f}%  {v['total_us']:12.1f} us  x{v['launches']:4d}  {k}\n")
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
