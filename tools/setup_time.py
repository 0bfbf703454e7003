"""bp_setup wall time, device vs host setup path, at given configs."""
import sys
import time

sys.path.insert(0, ".")
import paper_2109_04996_b200 as hx

for bp, p, d in [("bp5", 7, 25), ("bp5", 7, 66), ("bp5", 1, 465), ("bp3", 7, 31), ("bp6", 5, 48)]:
    for host in (False, True):
        t0 = time.perf_counter()
        pr = hx.setup(bp, degree=p, dims=(d, d, d), deform="sine", host_setup=host)
        t = time.perf_counter() - t0
        print(f"{bp} p={p} {d}^3 n={pr.n:,}: setup {'host' if host else 'device'} {t:.2f} s "
              f"(bp_setup {pr.setup_seconds:.2f} s)", flush=True)
        del pr
