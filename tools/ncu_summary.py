"""Summarise an ncu report: key raw metrics + top stalled SASS lines."""
import csv, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'sm__warps_active.avg.per_cycle_active', 'launch__grid_size', 'launch__block_size',
        'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__shared_mem_per_block_dynamic']
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:64s} {v[i][:60]} {u[i]}")
st = [(h[i], v[i]) for i in range(len(h)) if 'smsp__pcsamp_warps_issue_stalled' in h[i]
      and not h[i].endswith('not_issued')]
def f(x):
    try:
        return float(x.replace(',', ''))
    except ValueError:
        return 0.0
print("stall reasons:", ", ".join(f"{n.split('stalled_')[1]}={val}" for n, val in
                                  sorted(st, key=lambda t: -f(t[1]))[:8]))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    sc = h.index("Source")
    cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
    ci = [h.index(c) for c in cols]
    data = []
    for r in rows[2:]:
        if len(r) <= si:
            continue
        s = int(r[si]) if r[si].isdigit() else 0
        det = {cols[j][6:]: int(r[ci[j]]) for j in range(len(cols)) if r[ci[j]].isdigit() and int(r[ci[j]]) > 0}
        data.append((s, r[sc].strip(), det))
    tot = sum(d[0] for d in data) or 1
    for s, code, det in sorted(data, key=lambda t: -t[0])[:int(sys.argv[2])]:
        top = sorted(det.items(), key=lambda t: -t[1])[:2]
        print(f"{s:5d} {100*s/tot:4.1f}% {code[:58]:58s} {top}")
