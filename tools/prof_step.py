"""Small driver for ncu: BP5 p=7 25^3 setup, 3 operator applies, one 3-iteration PCG step."""
import sys
sys.path.insert(0, ".")
import argparse
import numpy as np
import torch
import paper_2109_04996_b200 as hx

ap = argparse.ArgumentParser()
ap.add_argument("--bp", default="bp5")
ap.add_argument("--degree", type=int, default=7)
ap.add_argument("--elems", type=int, default=25)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
prob = hx.setup(a.bp, degree=a.degree, dims=(a.elems,) * 3, deform="sine")
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, prob.size)).cuda()
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(3):
    prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
rep = prob.pcg_device(prob.rhs_device_ptr, x.data_ptr(), fixed_iterations=a.iters)
torch.cuda.synchronize()
print("ok", rep["iterations"])
