"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the
iteration on configs[0] and a small theta instance, the search direction and step lengths, a ragged task-graph
Cholesky (m = 300) and the virtual-rank distributed Cholesky (not product code)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import direction_G, gen_config  # noqa: E402
from paper_1310_6919_b200 import Handle  # noqa: E402
from paper_1310_6919_b200 import dist as D  # noqa: E402
from paper_1310_6919_b200.sdpc import scm_cholesky_virtual  # noqa: E402
from tests.helpers import scm_handle, small  # noqa: E402

dev = torch.device("cuda:0")
for inst in (gen_config(0), small("theta"), small("blockarrow")):
    h = Handle.from_instance(inst)
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    m = inst.m
    ld = m + (m & 1)
    Bt = torch.zeros((m, ld), dtype=torch.float64, device=dev)
    assert h.iteration(x, y, Bt, ld) == 0
    if inst.kind != "blockarrow":
        nnz = int(inst.colptr[-1])
        G = torch.from_numpy(direction_G(inst)).to(dev)
        g, dz = (torch.empty(m, dtype=torch.float64, device=dev) for _ in range(2))
        dY, dX = (torch.empty(nnz, dtype=torch.float64, device=dev) for _ in range(2))
        h.search_direction(x, G, 0.1, Bt, ld, g, dz, dY, dX)
        h.step_lengths(x, dX, y, dY)
    print("iteration ok", inst.name, flush=True)
m = 300
rng = np.random.default_rng(0)
G = rng.standard_normal((m, m + 3))
B = G @ G.T / (m + 3) + np.eye(m)
h = scm_handle(m)
Bt = torch.from_numpy(np.tril(B).T.copy()).to(dev)
assert h.scm_cholesky(Bt, m) == 0
P = 4
layouts = [D.Layout(m, P, r) for r in range(P)]
hs = [scm_handle(m, P, r) for r in range(P)]
lld = max(L.lld for L in layouts)
Bts = []
for L in layouts:
    b = torch.zeros((max(1, L.nloc), lld), dtype=torch.float64, device=dev)
    b[:L.nloc, :L.mloc] = torch.from_numpy(D.local_tiles_of(np.tril(B), L).T.copy()).to(dev)
    Bts.append(b)
assert scm_cholesky_virtual(hs, Bts, lld) == 0
torch.cuda.synchronize()
print("sanitize workload ok")
