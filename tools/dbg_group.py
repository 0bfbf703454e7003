import sys, threading, time
sys.path.insert(0, ".")
import torch
from paper_2109_04996_b200 import _core
N = 2
grid = tuple(_core.proc_grid(N, (4, 4, 4)))
gdims = tuple(4 * g for g in grid)
print("grid", grid, gdims, flush=True)
comms = _core.Communicator.group([0] * N)
def rank(r):
    print(r, "start", flush=True)
    if "torch" in sys.argv: torch.cuda.set_device(0)
    pr = _core.setup("bp5", 7, gdims, "sine", comm=comms[r], proc_grid=grid)
    print(r, "setup done", flush=True)
    x = torch.empty(pr.size, dtype=torch.float64, device="cuda:0")
    rep = pr.pcg_device(pr.rhs_device_ptr, x.data_ptr(), fixed_iterations=3, time_apply=False)
    print(r, "pcg done", rep["iterations"], flush=True)
ts = [threading.Thread(target=rank, args=(r,)) for r in range(N)]
[t.start() for t in ts]; [t.join() for t in ts]
print("ok", flush=True)
