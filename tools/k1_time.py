"""Time single operator applies (memset + K1) at a BP config, device events:
the number the ablation / variant A/B scripts compare (no PCG, so ablated
kernels that produce garbage are still timed)."""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2109_04996_b200 as hx

ap = argparse.ArgumentParser()
ap.add_argument("--bp", default="bp5")
ap.add_argument("--degree", type=int, default=7)
ap.add_argument("--elems", type=int, default=25)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--tag", default="")
a = ap.parse_args()
prob = hx.setup(a.bp, degree=a.degree, dims=(a.elems,) * 3, deform="sine")
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, prob.size)).cuda()
y = torch.empty_like(x)
s = torch.cuda.ExternalStream(prob.stream)
torch.cuda.synchronize()
for _ in range(5):
    prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(a.reps):
    prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / a.reps
m = 3 if a.bp in ("bp2", "bp4", "bp6") else 1
q = a.degree + (2 if a.bp in ("bp1", "bp2", "bp3", "bp4") else 1)
K = 6 if a.bp in ("bp3", "bp4", "bp5", "bp6") else 1
nL = (a.elems * a.degree + 1) ** 3
byt = 16 * m * nL + 8 * K * a.elems ** 3 * q ** 3
print(f"{a.tag} {a.bp} p={a.degree} {a.elems}^3: apply {us:.1f} us, {byt / us / 1e3:.0f} GB/s alg "
      f"({byt / us / 1e3 / 6551:.3f} of 6551)")
