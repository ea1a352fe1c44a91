"""One warm-up + one sdpc_iteration of a config (for ncu launch lists).  python tools/iter_once.py CFG"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from instances import gen_config  # noqa: E402
from paper_1310_6919_b200 import Handle  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
inst = gen_config(cfg)
h = Handle.from_instance(inst)
dev = torch.device("cuda:0")
x = torch.from_numpy(inst.xbar).to(dev)
y = torch.from_numpy(inst.y).to(dev)
m = inst.m
ld = m + (m & 1)
B = torch.zeros((m, ld), dtype=torch.float64, device=dev)
for _ in range(2):
    assert h.iteration(x, y, B, ld) == 0
torch.cuda.synchronize()
print("ok")
