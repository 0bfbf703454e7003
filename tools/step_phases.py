"""Phase timing of the fused PCG step kernel (measurement only): per-CTA
%globaltimer stamps at start, phase-1 end, after the grid barrier and at the
phase-2 end of one C3 bench-step iteration (odd and even)."""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2109_04996_b200 as hx
from paper_2109_04996_b200 import capi

lib = capi.lib()
prob = hx.setup("bp5", degree=7, dims=(25, 25, 25), deform="sine")
xs = torch.empty(prob.size, dtype=torch.float64, device="cuda")
buf = (ctypes.c_ulonglong * 4096)()
for it in (5, 6, 7, 8, 20):
    prob.pcg_device(prob.rhs_device_ptr, xs.data_ptr(), fixed_iterations=20, time_apply=False)
    torch.cuda.synchronize()
    lib.hxf_debug_step_timestamps(it, None)
    prob.pcg_device(prob.rhs_device_ptr, xs.data_ptr(), fixed_iterations=20, time_apply=False)
    torch.cuda.synchronize()
    lib.hxf_debug_step_timestamps(0, ctypes.cast(buf, ctypes.c_void_p))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 1024)[:, :148].astype(np.float64)
    t0 = a[0].min()
    a = (a - t0) / 1e3
    print(f"iteration {it}: start spread {a[0].max():.1f} us; phase 1 end min/med/max "
          f"{a[1].min():.1f}/{np.median(a[1]):.1f}/{a[1].max():.1f}; barrier out "
          f"{a[2].min():.1f}/{a[2].max():.1f}; phase 2 end {a[3].min():.1f}/{np.median(a[3]):.1f}/{a[3].max():.1f} us")
