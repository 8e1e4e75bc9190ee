"""cuBLAS DGEMM yardstick (library GEMM, measurement only): best-of and sustained FP64 TFLOP/s."""
import json, time, torch
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n**3 / best / 1e9
    print(f"cuBLAS DGEMM n={n}: {res[n]:.2f} TFLOP/s (best of 5)")
n = 8192; a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
torch.cuda.synchronize(); t0 = time.time(); k = 0
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"cuBLAS DGEMM n=8192 sustained: {2*n**3*k/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s over {k} calls")
