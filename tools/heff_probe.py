"""Two-site H_eff matvec (eigensolvers.hpp:15-64) at C4-like sizes: device call through the C-ABI
(host buffers, H2D/D2H included) vs the oracle restatement on the host.
Usage: python tools/heff_probe.py [chi] [D]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ttlab_oracle as O  # noqa: E402  (checker / CPU leg only)
from paper_2601_16734_b200 import ttlab as t  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 512
D = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rng = np.random.default_rng(1)
L = rng.standard_normal((D, chi, chi))
R = rng.standard_normal((D, chi, chi))
w1 = rng.standard_normal((D, 2, 2, D)) / np.sqrt(2 * D)
w2 = rng.standard_normal((D, 2, 2, D)) / np.sqrt(2 * D)
x = rng.standard_normal(chi * 4 * chi)
y = t.apply_effective_two_site(L, w1, w2, R, x)  # warm-up (context, allocations)
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    y = t.apply_effective_two_site(L, w1, w2, R, x)
gpu_ms = (time.perf_counter() - t0) / reps * 1e3
t0 = time.perf_counter()
ref = O.apply_effective_two_site(L, w1, w2, R, x)
cpu_ms = (time.perf_counter() - t0) * 1e3
err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
flops = 2 * D * chi * chi * 4 * chi * 2  # the two GEMM stages
print(f"chi={chi} D={D}: device call {gpu_ms:.2f} ms (host buffers, {flops / 1e9:.1f} GF in the GEMMs), "
      f"oracle {cpu_ms:.0f} ms, rel.err {err:.1e}")

# device-only matvec: device buffers (no host copies), CUDA events over `reps` chained calls, plus the
# per-class profile of one call (GEMM time -> achieved FP64 TF/s of the two GEMM stages)
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2601_16734_b200 import _lib  # noqa: E402

ctx = t.context()
dims = (C.c_int * 11)(D, D, D, 2, 2, 2, 2, chi, chi, chi, chi)
dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (L, w1, w2, R, x)]
yd = torch.empty(chi * 4 * chi, dtype=torch.float64, device="cuda")
stream = torch.cuda.Stream()  # a real stream shared by the library and the events (0 = the library's own)
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
args = [C.c_void_p(a.data_ptr()) for a in dev] + [C.c_void_p(yd.data_ptr())]
for _ in range(3):
    ctx.check(_lib.lib.ttg_apply_effective_two_site_dev(ctx.handle, _lib.TTG_F64, dims, *args))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record(stream)
for _ in range(reps):
    ctx.check(_lib.lib.ttg_apply_effective_two_site_dev(ctx.handle, _lib.TTG_F64, dims, *args))
e1.record(stream)
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1) / reps
ctx.profile_enable(True)
ctx.check(_lib.lib.ttg_apply_effective_two_site_dev(ctx.handle, _lib.TTG_F64, dims, *args))
prof = ctx.profile_read()
ctx.profile_enable(False)
g = prof["gemm"]
err = np.linalg.norm(yd.cpu().numpy() - ref) / np.linalg.norm(ref)
print(f"chi={chi} D={D}: device-only matvec {dev_ms:.3f} ms ({flops / dev_ms / 1e9:.1f} TF/s over the call); "
      f"GEMMs {g['ms']:.3f} ms for {g['flops'] / 1e9:.1f} GF = {g['flops'] / g['ms'] / 1e9:.1f} TF/s "
      f"({100 * g['flops'] / g['ms'] / 1e9 / 37.07:.0f}% of the 37.07 TF/s DMMA peak); mixing kernel "
      f"{prof['expand']['ms']:.3f} ms; rel.err {err:.1e}")
