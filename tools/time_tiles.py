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
