"""Microtest: a Triton-built (device-side tensormap.replace) TMA descriptor
vs the host-encoded one (cuTensorMapEncodeTiled) for the same 2-D f64 box."""
import ctypes as C

import torch
import triton
import triton.language as tl


@triton.jit
def k(out_ptr, in_ptr, M, N):
    desc = tl.make_tensor_descriptor(in_ptr, shape=[M, N], strides=[N, 1], block_shape=[8, 8])
    x = desc.load([2, 8])
    offs = tl.arange(0, 8)[:, None] * 8 + tl.arange(0, 8)[None, :]
    tl.store(out_ptr + offs, x)


ws = []


def alloc_fn(size, alignment, stream):
    t = torch.empty(size, device="cuda", dtype=torch.int8)
    ws.append(t)
    return t


triton.set_allocator(alloc_fn)
a = torch.arange(32 * 32, dtype=torch.float64, device="cuda").reshape(32, 32)
o = torch.empty(64, dtype=torch.float64, device="cuda")
h = k[(1,)](o, a, 32, 32)
torch.cuda.synchronize()
print("triton tma ok", o[:3].tolist(), "want", a[2, 8:11].tolist())
dev = ws[-1][:128].cpu().numpy().view("uint64")
print("triton desc:", " ".join(f"{v:016x}" for v in dev))

cu = C.CDLL("libcuda.so.1")
tm = (C.c_uint64 * 16)()
dims = (C.c_uint64 * 2)(32, 32)
strides = (C.c_uint64 * 1)(32 * 8)
box = (C.c_uint32 * 2)(8, 8)
es = (C.c_uint32 * 2)(1, 1)
for sw in (0, 2):
    r = cu.cuTensorMapEncodeTiled(tm, 8, 2, C.c_void_p(a.data_ptr()), dims, strides, box, es, 0, sw, 0, 0)
    print(f"host  desc sw{sw} (rc {r}):", " ".join(f"{v:016x}" for v in tm))
open("gpurun_out/tri.ptx", "w").write(h.asm["ptx"])
print("metadata:", {k: v for k, v in h.metadata._asdict().items() if k in ("num_ctas", "cluster_dims", "shared", "num_warps", "launch_cooperative_grid", "launch_pdl", "tmem_size", "global_scratch_size")} if hasattr(h.metadata, "_asdict") else h.metadata)
