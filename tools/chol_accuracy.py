"""Backward error of the SCM Cholesky per 128-tile (diagnostic): E = B - R R^T on the GPU (cuBLAS fp64)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from instances import gen_config
from paper_1310_6919_b200 import Handle

dev = torch.device("cuda:0")


def report(tag, B, R):
    Bs = torch.tril(B) + torch.tril(B, -1).T
    E = Bs - R @ R.T
    be = (torch.linalg.norm(E) / torch.linalg.norm(Bs)).item()
    m = B.shape[0]; T = (m + 127) // 128
    Et = torch.zeros(T, T, dtype=torch.float64)
    for i in range(T):
        for j in range(i + 1):
            Et[i, j] = torch.linalg.norm(E[i*128:(i+1)*128, j*128:(j+1)*128]).item()
    idx = torch.argsort(Et.flatten(), descending=True)[:8]
    top = [(int(x) // T, int(x) % T, float(Et.flatten()[x])) for x in idx]
    diag = float(torch.linalg.norm(torch.diagonal(Et)))
    print(f"{tag}: backward error {be:.3e}; diag-tile part {diag:.3e} of {float(torch.linalg.norm(Et)):.3e}; top tiles {top}", flush=True)
    # within the worst tile: error by column position
    i, j, _ = top[0]
    Ew = E[i*128:(i+1)*128, j*128:(j+1)*128].abs()
    print("  worst tile col maxima (every 8th):", [f"{v:.1e}" for v in Ew.max(0).values[::8].tolist()])
    print("  worst tile row maxima (every 8th):", [f"{v:.1e}" for v in Ew.max(1).values[::8].tolist()])


def chol(h, B, task_graph):
    h.set_cholesky_schedule(task_graph)
    m = B.shape[0]
    Bt = B.T.contiguous().clone()  # column-major storage
    assert h.scm_cholesky(Bt, m) == 0
    torch.cuda.synchronize()
    return torch.tril(Bt.T)


for cfg in [int(c) for c in (sys.argv[1:] or ["1"])]:
    inst = gen_config(cfg)
    h = Handle.from_instance(inst)
    m = inst.m
    x = torch.from_numpy(inst.xbar).to(dev); y = torch.from_numpy(inst.y).to(dev)
    h.factor_xinv(x)
    Bt = torch.zeros((m, m), dtype=torch.float64, device=dev)
    h.scm_build(y, Bt, m)
    B = torch.tril(Bt.T.contiguous())
    Bs = B + torch.tril(B, -1).T
    Rl = torch.linalg.cholesky(Bs)
    report(f"c{cfg} cusolver", B, Rl)
    report(f"c{cfg} dag", B, chol(h, B, True))
    report(f"c{cfg} multi-launch", B, chol(h, B, False))
    # a generic SPD matrix of the same size
    g = torch.Generator(device="cpu").manual_seed(1)
    G = torch.randn(m, m, generator=g, dtype=torch.float64).to(dev) / m ** 0.5
    S = G @ G.T + torch.eye(m, device=dev, dtype=torch.float64)
    S = torch.tril(S)
    report(f"random SPD m={m} dag", S, chol(h, S, True))
