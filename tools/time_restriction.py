"""Time the standalone element-restriction kernels (apply_g, apply_g_transpose,
gather_scalar, multiplicity; restriction.cpp:28-106) at C3 size on device
buffers: GB/s of their algorithmic bytes against the measured HBM peak."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2109_04996_b200 import capi

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6551.0
ctx = capi.Context(0)
for m, d, p in [(1, 25, 7), (3, 20, 7), (1, 44, 4)]:  # (HXF_BOX_RESTRICTION=0: the colour-class kernels)
    n1 = d * p + 1
    n_L, E, S = n1 ** 3, d ** 3, (p + 1) ** 3
    r = capi.ElemRestriction(ctx, p=p, m=m, num_elements=E, n_L=n_L, dims=(d, d, d))
    l = torch.rand(m * n_L, dtype=torch.float64, device="cuda")
    ev = torch.rand(m * E * S, dtype=torch.float64, device="cuda")
    es = torch.rand(E * S, dtype=torch.float64, device="cuda")

    def t(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / reps

    tg = t(lambda: r.apply_g(l))
    tt = t(lambda: r.apply_g_transpose(ev))
    ts = t(lambda: r.gather_scalar(es))
    bg = 8 * m * (n_L + E * S)      # read l once, write the E-vector
    bt = 8 * m * (E * S + n_L)      # read the E-vector, write l (zero-init included in the call)
    bs = 8 * (E * S + n_L)
    print(f"m={m} p={p} {d}^3 (E*S = {E * S:,}): apply_g {tg:.1f} us ({bg / tg / 1e3 / peak:.2f} of HBM), "
          f"apply_g_transpose {tt:.1f} us ({bt / tt / 1e3 / peak:.2f}), gather_scalar {ts:.1f} us "
          f"({bs / ts / 1e3 / peak:.2f})", flush=True)
    r.close()
