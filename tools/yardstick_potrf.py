"""Yardstick only (not product): cuSOLVER dpotrf (torch.linalg.cholesky, fp64) on an SPD m x m matrix,
CUDA events, to put the sdpc SCM Cholesky time in context.  usage: python tools/yardstick_potrf.py [m]"""
import sys
import torch

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
g = torch.Generator(device="cuda").manual_seed(0)
G = torch.randn(m, 256, dtype=torch.float64, device="cuda", generator=g)
B = G @ G.T / 256 + torch.eye(m, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.linalg.cholesky(B)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record()
    torch.linalg.cholesky(B)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"cuSOLVER dpotrf m={m}: {ms:.2f} ms, {m**3 / 3 / (ms * 1e-3) / 1e12:.2f} TF/s")

# cuBLAS DGEMM on the trailing-update shape (C -= A A^T with K = 256), yardstick for gemm_nt_kernel
for mm in (4096, 8192):
    A = torch.randn(mm, 256, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(mm, mm, dtype=torch.float64, device="cuda", generator=g)
    for _ in range(2):
        C.addmm_(A, A.T, alpha=-1.0)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        C.addmm_(A, A.T, alpha=-1.0)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cuBLAS DGEMM {mm}x{mm}x256: {ms:.3f} ms, {2 * mm * mm * 256 / (ms * 1e-3) / 1e12:.2f} TF/s")
