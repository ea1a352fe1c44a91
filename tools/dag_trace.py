"""Task-graph Cholesky diagnostics (not product code): per-task trace of one factorisation of a random
SPD m x m matrix, CTA utilisation, per-type task durations, the POTRF chain, and event timings of both
schedules.  python tools/dag_trace.py [m]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import scm_handle  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
G = torch.randn(m, 256, dtype=torch.float64, device=dev, generator=g)
ld = m + (m & 1)   # even ld: the task-graph kernel needs 16-byte staging
B0 = torch.zeros((m, ld), dtype=torch.float64, device=dev)
B0[:, :m] = G @ G.T / 256 + torch.eye(m, dtype=torch.float64, device=dev)
del G
B = B0.clone()
h = scm_handle(m)


def timed(sched, reps=3):
    h.set_cholesky_schedule(sched)
    ts = []
    for r in range(reps + 1):
        B.copy_(B0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert h.scm_cholesky(B, ld) == 0
        e1.record()
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return min(ts)


flops = m ** 3 / 3
for sched in (1, 0):
    t = timed(sched)
    print(f"schedule {sched}: {t:.3f} ms  {flops / t / 1e9:.2f} TF/s")

cap = 4_000_000
h.set_cholesky_schedule(1)
h.set_cholesky_trace(cap)
B.copy_(B0)
assert h.scm_cholesky(B, ld) == 0
tr, raw = h.get_cholesky_trace(cap)
tr = tr.astype(np.int64)
T = (m + 127) // 128
pst = raw[-16 * T:].astype(np.int64).reshape(T, 16)[:, :8]
h.set_cholesky_trace(0)
typ = tr[:, 0] >> 60
k = (tr[:, 0] >> 32) & 0xffff
t0 = tr[:, 1] - tr[:, 1].min()
t1 = tr[:, 2] - tr[:, 1].min()
cta = (tr[:, 3] >> 32) & 0xffff
nsteps = tr[:, 3] >> 48
smid = tr[:, 3] & 0xffffffff
chain_sms = np.unique(smid[typ == 1])
print("chain SMs (ran POTRF):", chain_sms.tolist())
span = t1.max()
ncta = len(np.unique(cta))
busy = (t1 - t0).sum()
# per-CTA gaps between the end of a task and the start of the next (notify + pop + barriers)
gaps = []
for c in np.unique(cta):
    idx = np.where(cta == c)[0]
    idx = idx[np.argsort(t0[idx])]
    g = t0[idx[1:]] - t1[idx[:-1]]
    gaps.append(g)
gaps = np.concatenate(gaps) / 1e3 if gaps else np.zeros(1)
print(f"inter-task gap per CTA: mean {gaps.mean():.2f} us  p50 {np.median(gaps):.2f}  p90 {np.percentile(gaps, 90):.2f}")
print(f"tasks {len(tr)}  span {span / 1e6:.3f} ms  CTAs {ncta}  utilisation {busy / (span * ncta):.3f}")
u = typ == 3
print(f"update tasks {u.sum()}, steps applied {nsteps[u].sum()}, mean steps/task {nsteps[u].mean():.2f}, "
      f"histogram {np.bincount(nsteps[u])[1:].tolist()}")
for ty, nm in ((1, "POTRF"), (2, "TRSM"), (3, "UPD")):
    d = (t1 - t0)[typ == ty] / 1e3
    if len(d):
        print(f"  {nm:5s} n={len(d):7d} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}"
              f"  max {d.max():7.2f}  total {d.sum() / 1e3:8.2f} ms")
pot = np.where(typ == 1)[0]
pot = pot[np.argsort(k[pot])]
ps, pe = t0[pot] / 1e3, t1[pot] / 1e3
gaps = ps[1:] - pe[:-1]
print(f"POTRF chain: first start {ps[0]:.1f} us, last end {pe[-1]:.1f} us; POTRF-to-next-POTRF gap mean {gaps.mean():.1f} us"
      f" p50 {np.median(gaps):.1f} max {gaps.max():.1f}")
ends = np.diff(pe)
print(f"chain step (POTRF end to next POTRF end): mean over the last 30 steps {ends[-30:].mean():.1f} us, "
      f"last 40 {ends[-40:].mean():.1f} us, all {ends.mean():.1f} us")
for kk in list(range(0, len(pot), max(1, len(pot) // 12))):
    print(f"  k={kk:4d} potrf [{ps[kk]:9.1f}, {pe[kk]:9.1f}] us")
# utilisation over time (10 bins)
bins = np.linspace(0, span, 11)
for b in range(10):
    lo, hi = bins[b], bins[b + 1]
    ov = np.clip(np.minimum(t1, hi) - np.maximum(t0, lo), 0, None).sum()
    print(f"  [{lo / 1e6:6.2f}, {hi / 1e6:6.2f}] ms busy {ov / ((hi - lo) * ncta):.3f}")

names = ["load", "p0", "p1", "p2", "p3", "Lstore", "Linv"]
d = np.diff(pst[:-1], axis=1) / 1e3
print("POTRF phases (us, mean over k < T-1): " + "  ".join(f"{nm} {v:.1f}" for nm, v in zip(names, d.mean(axis=0))))

# the panel chain step by step in the tail: POTRF(k) end -> TRSM(k+1, k, *) -> UPD(k+1, k+1, k, *) -> POTRF(k+1)
ii = (tr[:, 0] >> 16) & 0xffff
jj = tr[:, 0] & 0xffff
rows = []
for kk in range(max(0, T - 31), T - 1):
    pe_k = t1[(typ == 1) & (k == kk)]
    ts = np.where((typ == 2) & (k == kk) & (ii == kk + 1))[0]
    us = np.where((typ == 3) & (ii == kk + 1) & (jj == kk + 1) & (k + nsteps - 1 == kk))[0]
    pn = t0[(typ == 1) & (k == kk + 1)]
    if len(pe_k) and len(ts) and len(us) and len(pn):
        rows.append([t0[ts].min() - pe_k[0], (t1[ts] - t0[ts]).max(), t0[us].min() - t1[ts].max(),
                     (t1[us] - t0[us]).max(), pn[0] - t1[us].max(),
                     (t1[(typ == 1) & (k == kk + 1)] - pn)[0]])
if rows:
    r = np.array(rows) / 1e3
    nm = ["POTRF->TRSM gap", "TRSM", "TRSM->UPD gap", "UPD(diag)", "UPD->POTRF gap", "POTRF"]
    print("tail chain (us, mean over the last %d steps): " % len(r) + "  ".join(f"{a} {b:.1f}" for a, b in zip(nm, r.mean(0))))
