"""Time standalone operator applies (CUDA events) at C3; honours HXF_ABLATE.
Usage: python tools/time_apply.py [bp] [degree] [elems]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2109_04996_b200 as hx

bp = sys.argv[1] if len(sys.argv) > 1 else "bp5"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 7
d = int(sys.argv[3]) if len(sys.argv) > 3 else 25
prob = hx.setup(bp, degree=p, dims=(d, d, d), deform="sine")
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, prob.size)).cuda()
y = torch.empty_like(x)
st = torch.cuda.ExternalStream(prob.stream)
torch.cuda.synchronize()
for _ in range(5):
    prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 30
e0.record(st)
for _ in range(reps):
    prob.apply_device(x.data_ptr(), y.data_ptr(), prob.stream)
e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
print(f"{bp} p={p} {d}^3 apply {us:.1f} us  {prob.n / us / 1e3:.2f} GDOF/s")
