"""One process per rank, CUDA IPC mailboxes (the --gpus N layout, here two
processes sharing one GPU): the partitioned solve's interface exchange and
dot all-reduce run as peer-store kernels across processes, bootstrapped over
torch.distributed (gloo), and must reproduce the single-domain solve."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = r"""
import json, os, sys
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, os.environ["HXF_ROOT"])
from paper_2109_04996_b200 import _core, dist as hdist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
bp, p, dims = os.environ["HXF_CASE_BP"], int(os.environ["HXF_CASE_P"]), tuple(int(v) for v in os.environ["HXF_CASE_DIMS"].split(","))
m = 3 if bp in ("bp2", "bp4", "bp6") else 1
grid = tuple(_core.proc_grid(world, dims))
cap = max(hdist.p2p_capacity(_core.subdomain(dims, world, r).dims, p, m) for r in range(world))
comm = hdist.p2p_communicator(0, cap)
pr = _core.setup(bp, p, dims, "sine", comm=comm, proc_grid=grid)
ids = _core.global_node_ids(pr.subdomain, p)
nG = (dims[0] * p + 1) * (dims[1] * p + 1) * (dims[2] * p + 1)
x = np.random.default_rng(11).uniform(-1, 1, m * nG)
idx = np.concatenate([c * nG + ids for c in range(m)])
y = pr.apply(x[idx])
_, rep = pr.solve(tol=1e-8, fixed_iterations=10)
out = {"ids": idx.tolist(), "y": y.tolist(), "hist": rep["residual_history"].tolist(),
       "iters": rep["iterations"]}
with open(os.environ["HXF_OUT"] + f".{rank}", "w") as f:
    json.dump(out, f)
dist.barrier()
"""


@pytest.mark.parametrize("bp,p,dims,nproc", [("bp5", 4, (4, 3, 2), 2), ("bp5", 7, (4, 4, 2), 4),
                                             ("bp6", 5, (4, 2, 2), 2)])
def test_ipc_exchange_across_processes(tmp_path, bp, p, dims, nproc):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = {**os.environ, "HXF_ROOT": str(ROOT), "HXF_OUT": str(tmp_path / "out"),
           "PYTHONPATH": str(ROOT), "HXF_CASE_BP": bp, "HXF_CASE_P": str(p),
           "HXF_CASE_DIMS": ",".join(str(d) for d in dims)}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29533 + nproc), str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    sys.path.insert(0, str(ROOT))
    import oracle
    from paper_2109_04996_b200 import _core

    g = _core.setup(bp, p, dims, "sine")
    x = np.random.default_rng(11).uniform(-1, 1, g.size)
    y_g = g.apply(x)
    _, rep_g = g.solve(tol=1e-8, fixed_iterations=10)
    for rank in range(nproc):
        o = json.loads((tmp_path / f"out.{rank}").read_text())
        ids = np.asarray(o["ids"])
        assert oracle.rel_max_diff(y_g[ids], np.asarray(o["y"])) <= 1e-12
        assert o["iters"] == 10
        assert oracle.rel_max_diff(rep_g["residual_history"], np.asarray(o["hist"])) <= 1e-10
