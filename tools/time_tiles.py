"""Per-kernel latency of the SCM Cholesky building blocks (diagonal factorisation via
sdpc_potrf_tile, panel solve, trailing update), CUDA events over repeated launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import scm_handle  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


dev = torch.device("cuda:0")
for nb in (128, 256):
    h = scm_handle(nb)
    rng = np.random.default_rng(0)
    G = rng.standard_normal((nb, nb + 8))
    B0 = torch.from_numpy(G @ G.T / nb + np.eye(nb)).to(dev)
    Bt = B0.clone()
    inv = torch.zeros(2 * 128 * 128, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)

    def run():
        Bt.copy_(B0)
        h.potrf_tile(Bt, nb, nb, inv, info)
    t = timeit(run)
    tc = timeit(lambda: Bt.copy_(B0))
    print(f"potrf_tile nb={nb}: {t - tc:.1f} us per call (copy {tc:.1f} us excluded)")

# standalone trailing-update GEMM (the dominant kernel) through sdpc_update_tiles on a 1 x 1 grid:
# C[k1:, k1:] (lower) -= P P^T with K = 256
for m in (4096, 10000):
    h = scm_handle(m)
    C = torch.zeros((m, m), dtype=torch.float64, device=dev)      # column-major view: C[j, i]
    P = torch.randn((256, m), dtype=torch.float64, device=dev)      # panel: row r = global row 256 + r
    k1 = 256
    t = timeit(lambda: h.update_tiles(C, m, P, m, k1, 256), reps=10)
    r = m - k1
    fl = r * (r + 1) * 256.0
    print(f"update_tiles m={m} K=256: {t:.1f} us, {fl / (t * 1e-6) / 1e12:.2f} TF/s")
