import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from tests.helpers import scm_handle
dev = torch.device("cuda:0")
for m in (256, 384, 1000):
  for fill in (0.0, float("nan")):
    h = scm_handle(m)
    rng = np.random.default_rng(m * 7)
    G = rng.standard_normal((m, m + 8))
    Bh = G @ G.T / (m + 8) + 0.5 * np.eye(m)
    Bt = torch.full((m, m), fill, dtype=torch.float64, device=dev)
    Bt[:, :m] = torch.from_numpy(np.tril(Bh).T.copy()).to(dev)
    if fill != 0.0:
        Bt = torch.where(torch.from_numpy(np.tril(np.ones((m, m))).T.copy()).to(dev) > 0, Bt, torch.tensor(fill, dtype=torch.float64, device=dev))
    info = h.scm_cholesky(Bt, m)
    R = np.tril(Bt.T.cpu().numpy())
    Ro = np.linalg.cholesky(Bh)
    T = (m + 127) // 128
    errs = [[float(np.abs(R[128*i:128*i+128, 128*j:128*j+128] - Ro[128*i:128*i+128, 128*j:128*j+128]).max()) for j in range(i + 1)] for i in range(T)]
    print(m, fill, info, errs)
