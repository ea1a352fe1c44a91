"""One task-graph (or multi-launch) SCM Cholesky of a random SPD m x m matrix (for ncu; not product code).
python tools/chol_once.py [m] [schedule] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import scm_handle  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
sched = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
ld = m + (m & 1)
G = torch.randn(m, 256, dtype=torch.float64, device=dev, generator=g)
B0 = torch.zeros((m, ld), dtype=torch.float64, device=dev)
B0[:, :m] = G @ G.T / 256 + torch.eye(m, dtype=torch.float64, device=dev)
del G
B = B0.clone()
h = scm_handle(m)
h.set_cholesky_schedule(sched)
for _ in range(reps):
    B.copy_(B0)
    assert h.scm_cholesky(B, ld) == 0
torch.cuda.synchronize()
print("ok")
