"""Every BASELINE.json workload on one B200: ms per iteration split into
construction and update, each as an absolute time and as a fraction of its
roofline, with the reference's CPU Engine timed on the same host in the same
run (north star "For every workload, report ...").

    python tools/workloads.py [--out gpurun_out/workloads.json] [--quick]

Multi-GPU configurations run as SHARD EMULATION on the one GPU: an engine in
external-exchange mode (world = G, rank 0, no NCCL) builds exactly rank 0's
ant shard (m/G ants; the ants are keyed by their global id) and runs the
replicated update.  Construction and update times are therefore the per-GPU
device times of a G-GPU run; the NCCL exchange itself cannot be timed on a
one-GPU box and is reported as bytes moved, its time as a labelled model.

Rooflines:
  construction (roulette): B_c = m_local*(n-1)*n*4 bytes (one fp32 row per
      ant-step) over the live-measured L2 row-staging peak;
  construction (nn):       m_local*(n-1)*(nn*(8+4)) list bytes + one fp64 row
      (n*8) per argmax-fallback step, over the same L2 peak (the lists are
      L2-resident; the fallback rows stream from HBM at 10k);
  update (accumulate, G=1): evaporate 16*n*P + deposit 2*m*n red.f64 (8 B each)
      + tours 4*m*(n+1) + choice epilogue (8+4+8+S)*n*P, over HBM peak;
  update (accumulate, G>1): k_rows<DELTA> (8+8+8+8+4+8+S)*n*P (the local
      red.f64 deposit runs in the construction phase; shard emulation runs
      the fp64 external-exchange kernel — the NCCL path's k_delta_pack +
      k_rows<DELTA32> are timed separately by tools/pack_cost.py);
  update (gather):         (8+8+4+8+S)*n*P + 16*m*n + 8*m, over HBM peak
      (G > 1: the row-sharded fold of n/G rows + the apply of all rows,
      timed around aco_gpu_fold + aco_gpu_update);
  S = 4 for the roulette's fp32 stream, 0 for nn; nn adds the top-K rebuild's
      8*n*P re-read of the choice rows.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def l2_and_hbm_peaks(device=0):
    import bench

    bw = bench.measure_l2_read_bw(device)
    peaks = bench.load_peaks()
    return {"l2_gbs": bw["l2_read_gbs"], "l2_rows_gbs": bw["l2_rows_gbs"],
            "l2_cg_gbs": bw["l2_cg_gbs"],
            "hbm_gbs": peaks.get("hbm_gbs") or bw["hbm_read_gbs"],
            "hbm_source": "MEASURED_PEAKS.json hbm_gbs" if peaks.get("hbm_gbs")
            else "live 2 GiB read (libaco_probe.so)"}


def time_engine(aco, torch, prob, n, m, selection, deposit, G, iters, warmup, nn=30, wire=0):
    cfg = aco.RunConfig(params=aco.Parameters(m=m, seed=1, nn=nn),
                        selection=aco.SelectionStrategy(aco.Selection(selection)),
                        deposit=aco.DepositStrategy(aco.Deposit(deposit)),
                        world=G, rank=0, wire=aco.Wire(wire))
    if wire == 2 and G > 1:
        # the fixed-point wire has no external-exchange mode: one GPU's share
        # is emulated by a one-GPU colony of ceil(m/G) ants (the same kernels
        # on the same number of ants; its own records only)
        cfg.world = 1
        cfg.params.m = -(-(m or n) // G)
    eng = aco.Engine(prob, cfg)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sp = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda")
    recs = []
    rowshard = G > 1 and deposit != 0  # row-sharded gather: construct, fold, update
    if rowshard:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from test_gpu_sharded import DevArray

        xb = eng.exchange_buffers()
        S = xb["S"]
        tabs = [torch.as_tensor(DevArray(xb[k], (G, n, S), "<i4"), device="cuda") for k in ("succ", "pred")]
        inv = torch.as_tensor(DevArray(xb["inv"], (G, S), "<f8"), device="cuda")
    for i in range(warmup + iters):
        with torch.cuda.stream(sp):
            flush.fill_(i & 0xFF)
        if not rowshard:
            r = eng.run_iteration()
        else:
            # rank 0's shard; the other ranks' succ/pred/1/C_k blocks stand in
            # as copies of rank 0's (same duplicate statistics), so the fold
            # of rank 0's n/G rows and the apply run on realistic data
            r = eng.construct()
            torch.cuda.synchronize()
            for t in tabs + [inv]:
                for g in range(1, G):
                    t[g].copy_(t[0])
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(sp):
                a.record(sp)
            eng.fold()
            eng.update()
            with torch.cuda.stream(sp):
                b.record(sp)
            b.synchronize()
            r.update_ms = a.elapsed_time(b)  # fold + apply, incl. two host calls
        if i >= warmup:
            recs.append(r)
    torch.cuda.synchronize()
    out = {
        "m_local": eng.ant_end - eng.ant_begin,
        "construct_ms": statistics.median(r.construct_ms for r in recs),
        "construct_kernel_ms": statistics.median(r.construct_kernel_ms for r in recs),
        "update_ms": statistics.median(r.update_ms for r in recs),
        "choice_ms": statistics.median(r.choice_ms for r in recs),
        "fallback_steps_per_iter": statistics.mean(r.fallbacks for r in recs),
        "best_length_last": recs[-1].best_length,
        "kernel": eng.describe(),
        "iterations": iters,
    }
    out["ms_per_iter"] = out["construct_ms"] + out["update_ms"]
    eng.close()
    del flush
    return out


def cpu_reference(n, m, selection, deposit, iters, nn=30):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import RefEngine, synth_coords  # cpu baseline leg only

    xs, ys = synth_coords(n)
    t0 = time.time()
    eng = RefEngine(xs, ys, m=m, nn=nn, seed=1, selection=selection, deposit=deposit, workers=0)
    create = time.time() - t0
    recs = [eng.run_iteration() for _ in range(iters)]
    return {"construct_ms": statistics.mean(r["construct_ms"] for r in recs),
            "update_ms": statistics.mean(r["update_ms"] for r in recs),
            "ms_per_iter": statistics.mean(r["construct_ms"] + r["update_ms"] for r in recs),
            "cores": eng.workers, "iterations": iters, "create_s": round(create, 2),
            "kind": "reference (oracle/_ref: proj/include/aco compiled unmodified, -O3)"}


def rooflines(res, n, m_total, selection, deposit, nn, peaks):
    P = (n + 31) // 32 * 32
    ml = res["m_local"]
    if selection == 1:
        b_c = ml * (n - 1) * nn * (8 + 4) + res["fallback_steps_per_iter"] * n * 8
    else:
        b_c = ml * (n - 1) * n * 4
    s32 = 4 if selection == 0 else 0          # the fp32 streamed copy (roulette only)
    topk = 8 * n * P if selection == 1 else 0  # k_row_topk re-reads the choice rows
    if deposit == 0 and res.get("G", 1) > 1:   # k_rows<DELTA>: tau, delta r/w, dist, choice
        b_u = (8 + 8 + 8 + 8 + 4 + 8 + s32) * n * P + topk
    elif deposit == 0:                         # evaporate + red.f64 + k_rows<CHOICE>
        b_u = 16 * n * P + 2 * m_total * n * 8 + 4 * m_total * (n + 1) + (8 + 4 + 8 + s32) * n * P + topk
    elif res.get("G", 1) > 1:                  # row-sharded: fold n/G rows, apply all rows
        B = -(-n // res["G"])
        b_u = 8 * m_total * B + 8 * B * P + (8 + 8 + 8 + 4 + 8 + s32) * n * P + topk
    else:                                      # k_rows gather: tau r/w, dist, choice + succ/pred
        b_u = (8 + 8 + 4 + 8 + s32) * n * P + 16 * m_total * n + 8 * m_total + topk
    c_gbs = b_c / (res["construct_kernel_ms"] * 1e-3) / 1e9
    u_gbs = b_u / (res["update_ms"] * 1e-3) / 1e9
    return {
        "construct": {"bytes": int(b_c), "achieved_gbs": round(c_gbs, 1), "bound": "l2",
                      "peak_gbs": peaks["l2_gbs"], "frac": round(c_gbs / peaks["l2_gbs"], 4)},
        "update": {"bytes": int(b_u), "achieved_gbs": round(u_gbs, 1), "bound": "hbm",
                   "peak_gbs": peaks["hbm_gbs"], "frac": round(u_gbs / peaks["hbm_gbs"], 4)},
    }


def exchange_model(n, m_total, G, deposit, wire_kind=0, selection=0, nn=30, records=0):
    """Bytes each GPU sends per iteration over NVLink and a labelled time model
    (ring all-reduce / all-gather at 700 GB/s bus bandwidth; not measured).
    wire_kind: 0 fp64 (default), 1 fp32, 2 fixed64 (int64 sums; nn selection:
    compact n x nn slots + the non-list edge records)."""
    if G == 1:
        return None
    P = (n + 31) // 32 * 32
    if deposit == 0 and wire_kind == 2 and selection == 1:
        slots = n * nn * 8
        rec = G * records * 16  # every rank's records, all-gathered
        wire = 2 * (G - 1) / G * slots + (G - 1) / G * rec
        what = (f"ncclAllReduce(slots, {n}x{nn} u64) + ncclAllGather(records, "
                f"~{records} x 16 B per rank)")
    elif deposit == 0:
        esz = 4 if wire_kind == 1 else 8
        size = n * P * esz
        wire = 2 * (G - 1) / G * size
        what = f"ncclAllReduce(delta, {n}x{P} {['f64', 'f32', 'u64'][wire_kind]}, sum)"
    else:  # row-sharded gather
        S = -(-m_total // G)
        B = -(-n // G)
        wire = (G - 1) * (2 * B * S * 4 + S * 8 + B * P * 8)
        what = ("ncclSend/Recv(succ, pred row blocks) + ncclAllGather(1/C_k) + "
                "ncclAllGather(delta row blocks)")
    return {"collective": what, "bytes_per_gpu": int(wire),
            "modelled_ms": round(wire / 700e9 * 1e3, 4),
            "model": "bytes_per_gpu / 700 GB/s NVLink-5 bus bandwidth (not measured: 1-GPU box)"}


def _records(res):
    """nn + fixed64: non-list edges per shard ~ argmax fallbacks + one closing
    edge per ant (from the engine's describe())."""
    import re

    m = re.search(r"argmax_fallbacks=(\d+)", res.get("kernel", ""))
    return (int(m.group(1)) if m else 0) + res["m_local"]


WORKLOADS = [
    # name, n, m (0 = n), selection, deposits, G list, iterations, cpu iterations
    ("d198", 198, 0, 0, (0, 1), (1,), 10, 10),
    ("pr1002", 1002, 0, 0, (0, 1), (1,), 10, 2),
    ("pr2392", 2392, 0, 0, (0, 1), (1, 2, 4, 8), 10, 2),
    ("pr2392x8ants", 2392, 8 * 2392, 0, (0, 1), (1, 2, 4, 8), 5, 1),
    ("synth10k_nn30", 10000, 0, 1, (0,), (1, 8), 3, 1),
    # config 5 on the exact fixed-point wire: the sharded exchange is the
    # compact nn slots + records instead of the n^2 delta
    ("synth10k_nn30_fixed64", 10000, 0, 1, (0,), (1, 8), 3, 0),
]
WIRE = {"synth10k_nn30_fixed64": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "workloads.json"))
    ap.add_argument("--quick", action="store_true", help="fewer iterations, no CPU baseline")
    ap.add_argument("--only", default="")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_1101_2678_b200 import aco

    peaks = l2_and_hbm_peaks()
    report = {"peaks": peaks, "gpu": torch.cuda.get_device_name(0), "workloads": []}
    for name, n, m, sel, deps, Gs, iters, cpu_iters in WORKLOADS:
        if a.only and name not in a.only.split(","):
            continue
        m_total = m or n
        prob = aco.build_problem(aco.synthetic_instance(n))
        for dep in deps:
            for G in Gs:
                it = 2 if a.quick else iters
                t0 = time.time()
                wk = WIRE.get(name, 0)
                res = time_engine(aco, torch, prob, n, m, sel, dep, G, it, 2, wire=wk)
                res["G"] = G
                res["wall_s"] = round(time.time() - t0, 1)
                entry = {"workload": name, "n": n, "m": m_total, "G": G,
                         "selection": aco.selection_name(aco.Selection(sel)),
                         "deposit": aco.deposit_name(aco.Deposit(dep)), **res,
                         "roofline": rooflines(res, n, m_total, sel, dep, 30, peaks),
                         "wire": ["fp64", "fp32", "fixed64"][wk],
                         "exchange": exchange_model(n, m_total, G, dep, wk, sel, 30,
                                                    records=_records(res))}
                if G > 1:
                    entry["ants_per_s_job"] = round(m_total / (res["ms_per_iter"] * 1e-3), 1)
                print(json.dumps(entry), flush=True)
                report["workloads"].append(entry)
        if not (a.quick or a.no_cpu) and cpu_iters:
            # reference CPU: accumulate always; the O(n^4) gather family only at d198
            for dep in deps:
                if dep == 1 and n > 198:
                    continue
                t0 = time.time()
                ref = cpu_reference(n, m, sel, dep, cpu_iters)
                ref["wall_s"] = round(time.time() - t0, 1)
                entry = {"workload": name, "n": n, "m": m_total, "impl": "reference-cpu",
                         "deposit": aco.deposit_name(aco.Deposit(dep)), **ref}
                print(json.dumps(entry), flush=True)
                report["workloads"].append(entry)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
