"""Throughput sweep (BASELINE configs[4], SURVEY §8(d) C5 grid): GDOF/s of one
operator apply and per CG iteration vs p and DOFs per GPU, with the HBM
roofline fraction of each (algorithmic bytes / time / measured HBM peak).

Usage: python tools/sweep.py [--bp bp5] [--p 1-15] [--sizes 1e5,1e6,1e7]
       [--deform sine] [--out profiles/r1_sweep_bp5.md]
       [--records sweep.jsonl] [--csv sweep.csv] [--cpu [--cpu-iters 3]]
--cpu times the reference itself (oracle/_ref run_bench, min of 3 reps, all
host cores, --cpu-iters fixed CG iterations) at every point.
--records writes one reference BenchRecord JSON per point (bench.cpp:351-363,
P = 1 GPU) and --csv the reference's sweep CSV (bench.cpp:365-381, eta = 1 at
P = 1; multi-GPU rows come from bench.py --gpus N and
_core.scaling_summary).
Elements per axis come from SURVEY §8(d)'s C5 table: d chosen so that
n = m (d p - 1)^3 is closest to the target (constrained BPs)."""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

import paper_2109_04996_b200 as hx


def parse_range(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def sizes_for(bp, p, d):
    k = int(bp[2])
    m = 1 if k % 2 == 1 else 3
    q = p + 2 if k <= 4 else p + 1
    n1 = d * p + 1
    cons = k >= 3
    n = m * ((n1 - 2) ** 3 if cons else n1 ** 3)
    K = 6 if k >= 3 else 1
    ba = 16 * m * n1 ** 3 + 8 * K * d ** 3 * q ** 3
    return n, ba, ba + 88 * m * n1 ** 3


def flops_apply(bp, p, d):
    """Algorithmic FP64 flops of one fused apply: per element
    and component, BP5/6 12 P^4 + 15 P^3; BP3/4 4 (I + 3 q^4) + 15 q^3; BP1/2
    4 I + q^3, with I = q P^3 + q^2 P^2 + q^3 P (P = p+1)."""
    k = int(bp[2])
    m = 1 if k % 2 == 1 else 3
    P = p + 1
    q = p + 2 if k <= 4 else p + 1
    interp = q * P ** 3 + q * q * P * P + q ** 3 * P
    if k >= 5:
        f = 12 * P ** 4 + 15 * P ** 3
    elif k >= 3:
        f = 4 * (interp + 3 * q ** 4) + 15 * q ** 3
    else:
        f = 4 * interp + q ** 3
    return f * m * d ** 3


FP64_PEAK_TFS = 37.0  # DMMA m8n8k4 rate measured on this B200 (tools/micro/fp64_rate.cu)


def pick_d(bp, p, target):
    best = None
    for d in range(1, 2000):
        n = sizes_for(bp, p, d)[0]
        if best is None or abs(np.log(n / target)) < abs(np.log(sizes_for(bp, p, best)[0] / target)):
            best = d
        if n > 4 * target:
            break
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bp", default="bp5")
    ap.add_argument("--p", default="1-15")
    ap.add_argument("--sizes", default="1e5,1e6,1e7")
    ap.add_argument("--dims", default=None, help="fixed d (overrides --sizes)")
    ap.add_argument("--deform", default="sine")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--records", default=None)
    ap.add_argument("--csv", default=None)
    ap.add_argument("--cpu", action="store_true",
                    help="time the reference (oracle/_ref run_bench, all host cores) at each point")
    ap.add_argument("--cpu-iters", type=int, default=3)
    a = ap.parse_args()
    peak = json.load(open(ROOT / "MEASURED_PEAKS.json"))["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    rows = []
    targets = [None] if a.dims else [float(s) for s in a.sizes.split(",")]
    for p in parse_range(a.p):
        for tgt in targets:
            d = int(a.dims) if a.dims else pick_d(a.bp, p, tgt)
            n, bapply, bcg = sizes_for(a.bp, p, d)
            t0 = time.perf_counter()
            prob = hx.setup(a.bp, degree=p, dims=(d, d, d), deform=a.deform)
            tsetup = time.perf_counter() - t0
            st = torch.cuda.ExternalStream(prob.stream)
            x = torch.from_numpy(np.random.default_rng(99).uniform(-1, 1, prob.size)).cuda()
            y = torch.empty_like(x)
            xs = torch.empty_like(x)
            torch.cuda.synchronize()
            for _ in range(3):
                prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
            reps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
            e1.record(st)
            torch.cuda.synchronize()
            t_apply = e0.elapsed_time(e1) * 1e-3 / reps
            b = prob.rhs_device_ptr
            prob.pcg_device(b, xs.data_ptr(), fixed_iterations=a.iters, time_apply=False)
            best = float("inf")
            for _ in range(3):
                torch.cuda.synchronize()
                e0.record(st)
                prob.pcg_device(b, xs.data_ptr(), fixed_iterations=a.iters, time_apply=False)
                e1.record(st)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e-3)
            t_it = best / a.iters
            k1 = prob.pcg_device(b, xs.data_ptr(), fixed_iterations=a.iters,
                                 time_apply=True)["apply_time_seconds"] / a.iters
            row = dict(bp=a.bp, p=p, d=d, n=n, apply_us=t_apply * 1e6,
                       apply_gdofs=n / t_apply / 1e9, apply_frac=bapply / t_apply / 1e9 / peak,
                       k1_us=k1 * 1e6, k1_frac=bapply / k1 / 1e9 / peak,
                       cg_us=t_it * 1e6, cg_gdofs=n / t_it / 1e9,
                       cg_frac=bcg / t_it / 1e9 / peak, setup_s=tsetup,
                       k1_tflops=flops_apply(a.bp, p, d) / k1 / 1e12)
            if a.cpu:
                import os

                import oracle
                cores = os.cpu_count() or 1
                t0 = time.perf_counter()
                ref = oracle.run_bench_reference(a.bp, p, (d, d, d), cores, a.cpu_iters, a.deform)
                row.update(cpu_gdofs=ref["dofs_rate"] / 1e9, cpu_cores=cores,
                           cpu_wall_s=time.perf_counter() - t0)
            q = p + 2 if int(a.bp[2]) <= 4 else p + 1
            row["record"] = dict(bp=a.bp, p=p, q=q, E=d ** 3, n=n, P=1, iterations=a.iters,
                                 seconds=best, dofs_rate=n * a.iters / best, n_per_rank=float(n))
            rows.append(row)
            print(json.dumps({k: v for k, v in row.items() if k != "record"}), flush=True)
            del prob, x, y, xs
            torch.cuda.empty_cache()
    from paper_2109_04996_b200 import _core
    if a.records:
        with open(a.records, "w") as f:
            for r in rows:
                f.write(_core.bench_record_json(r["record"]) + "\n")
    if a.csv:
        srows = [dict(record=r["record"], T_1=r["record"]["seconds"], T_P=r["record"]["seconds"],
                      eta=1.0) for r in rows]
        with open(a.csv, "w") as f:
            f.write(_core.scaling_summary(srows)["csv"])
    if a.out:
        with open(a.out, "w") as f:
            f.write(f"# {a.bp} throughput sweep ({a.deform} box, {a.iters} fixed CG iterations, "
                    f"HBM peak {peak} GB/s measured)\n\n")
            cpu = a.cpu and rows
            f.write("| p | d | n (DOFs) | apply us | apply GDOF/s | apply roof | K1 us | K1 roof "
                    "| K1 FP64 TF/s (of 37) | CG us/iter | CG GDOF/s | CG roof |" +
                    (f" ref CPU GDOF/s ({rows[0]['cpu_cores']} thr) | CG speed-up |" if cpu else "") +
                    "\n|---|---|---|---|---|---|---|---|---|---|---|---|" + ("---|---|" if cpu else "") + "\n")
            for r in rows:
                f.write(f"| {r['p']} | {r['d']} | {r['n']:,} | {r['apply_us']:.1f} | "
                        f"{r['apply_gdofs']:.2f} | {r['apply_frac']:.2f} | {r['k1_us']:.1f} | "
                        f"{r['k1_frac']:.2f} | {r['k1_tflops']:.1f} ({r['k1_tflops'] / FP64_PEAK_TFS:.2f}) | "
                        f"{r['cg_us']:.1f} | {r['cg_gdofs']:.2f} | "
                        f"{r['cg_frac']:.2f} |" +
                        (f" {r['cpu_gdofs']:.4f} | {r['cg_gdofs'] / r['cpu_gdofs']:.0f}x |" if cpu else "") +
                        "\n")


if __name__ == "__main__":
    main()
