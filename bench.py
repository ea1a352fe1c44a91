#!/usr/bin/env python
"""Benchmark of one MC-PDIPM SCM iteration (build + Cholesky) on B200.

BASELINE.json metric: "SCM build+Cholesky s/iter, B-entries/s, % HBM/FP64 roofline at 1/2/4/8 B200".
One step = sdpc_iteration: (a1) Algorithm 1 and (a2) chol(Y) concurrently, then (b) solves,
(c) accumulate, (d) SCM Cholesky, on fixed seeded synthetic inputs.  value = B-entries/s
= m(m+1)/2 / (s/iter), summed over ranks.  Default workload: configs[1] (max-cut on the 100x100
torus, n = m = 10,000), the configuration the metric is quoted on that fits one GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/, the only other place bench.py executes it) on the host
cores: Algorithm 1, the Y factorisation, the SCM columns in a first-come-first-served process pool
(the paper's Algorithm 2) and LAPACK potrf at the true m.  Configs 0-2 build the full B;
configs 3-4 fit t_fixed + t_col |cols| on two column samples and extrapolate t_col only.  The same
measurement is the `cpu_baseline` object of our line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SCM build+Cholesky s/iter, B-entries/s, % HBM/FP64 roofline at 1/2/4/8 B200"
CONFIG_TEXT = {
    0: "configs[0]: max-cut SDP, 10x10 torus, n=m=100, MD order",
    1: "configs[1]: spin-glass max-cut SDP, 100x100 torus, n=m=10000, ND order",
    2: "configs[2]: theta max-clique SDP, 60x60 torus, n=3600, m=7201, MD order",
    3: "configs[3]: block-arrow SDP, n=20200, m=5000, identity order",
    4: "configs[4]: max-cut SDP, 200x200 torus, n=m=40000, ND order",
    5: "NEXT 4 (not a BASELINE config): max-cut SDP on the 18x18x18 3D torus (SpinGlass18 shape), n=m=5832, 3D ND",
    6: "NEXT 4 (not a BASELINE config): max-cut SDP on the 25x25x25 3D torus (SpinGlass25 shape), n=m=15625, 3D ND",
}
# Nominal B200 ratio FP64-tensor / BF16-dense (45 / 2250 TFLOP/s, /opt/skills guides) applied to the
# measured bf16 peak (MEASURED_PEAKS.json) -> FP64 tensor peak for the roofline.
FP64_OVER_BF16 = 45.0 / 2250.0
FALLBACK_BF16 = dict(burst=1590.0, sustained=1400.0)   # B200_PROFILING.md fallback
FALLBACK_HBM = 6650.0
# ncu --set full of one chol_dag_kernel launch on a 10,000^2 SPD matrix (configs[1]'s m): dram__bytes_read.sum +
# dram__bytes_write.sum per algorithmic flop (m^3/3), scaled to the step's m^3/3 (profiles/r02/ncu/).
DAG_BYTES_PER_FLOP = (4.289942e9 + 4.113768e9) / (1e4 ** 3 / 3.0)
DAG_TRAFFIC_SOURCE = ("profiles/r02/final3/ncu_dag_full.txt: 4.29 GB read + 4.11 GB written by one chol_dag_kernel launch "
                      "at m = 10,000 (3.33e11 flops), scaled by the step's m^3/3")


def solve_flops(st, inst, truncated):
    """Algorithmic flops of the multi-RHS solves (b) for the X-hat and the Y^{-1} factor:
    per RHS p, forward over the etree reach of p (2 (cc_j + 1) per column j on the path), D scaling (n),
    backward over all of E (2 nnz(E)) or, with the max-cut truncation, over E[p:, p:].  RHS = the vertices
    the constraints touch (elimination ids).  Computed on the host from the structure."""
    import numpy as np
    n = int(st["n"])
    colptr = np.asarray(st["colptr"], dtype=np.int64)
    parent = np.asarray(st["parent"], dtype=np.int64)
    perm = np.asarray(st["perm"], dtype=np.int64)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    w = np.diff(colptr).astype(np.float64)                   # cc_j + 1
    rows = np.concatenate([inst.a_row[inst.a_ptr[1]:], inst.a_col[inst.a_ptr[1]:]])
    rhs = np.zeros(n, dtype=bool)
    rhs[iperm[np.unique(rows)]] = True
    # reach(p) = etree path p -> root; count of RHS below each node = RHS in its subtree (children < parent)
    cnt = rhs.astype(np.float64)
    for j in range(n):
        if parent[j] >= 0:
            cnt[parent[j]] += cnt[j]
    fwd = 2.0 * float(np.sum(cnt * w))
    nnz = float(colptr[-1])
    nr = float(rhs.sum())
    if truncated:
        # sum over RHS p of nnz(E[p:, p:]) = sum_j (number of RHS p <= j) (cc_j + 1)
        bwd = 2.0 * float(np.sum(np.cumsum(rhs) * w))
    else:
        bwd = 2.0 * nnz * nr
    per_factor = fwd + bwd + n * nr
    return per_factor, per_factor


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return dict(bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    hbm=d["hbm_gbs"], src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(bf16=FALLBACK_BF16["burst"], bf16_sus=FALLBACK_BF16["sustained"], hbm=FALLBACK_HBM,
                    src="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def entries(m):
    return m * (m + 1) / 2.0


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    if world > 1:
        return run_ours_dist(args, rank, world, local_rank)
    import numpy as np
    import torch

    import __graft_entry__
    from instances import gen_config

    __graft_entry__.build()
    from paper_1310_6919_b200 import Handle, fp64_peak

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    inst = gen_config(args.config, seed=args.seed)
    n, m = inst.n, inst.m
    h = Handle.from_instance(inst, device=local_rank)
    st = h.get_structure()
    assert np.array_equal(st["rowind"], inst.rowind), "library E differs from the generator's E"
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    ld = m + (m & 1)
    Bt = torch.empty((m, ld), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()

    def step():
        # sdpc_iteration: (a1) || (a2) on two streams, then (b), (c), (d); one host sync
        info = h.iteration(x, y, Bt, ld, stream)
        assert info == 0

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = h.launch_count()
    times, phases, ktimes = [], [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)                      # L2 flush between timed iterations (not timed)
            ev0.record(stream)
            step()
            ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            phases.append(h.phase_times())
            ktimes.append(h.kernel_times())
    torch.cuda.synchronize()
    launches = h.launch_count() - l0
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()

    # NEXT row 2 (not part of the metric): the SCE B dz = g with the factor just computed
    g_rhs = torch.ones((1, ld), dtype=torch.float64, device=dev)
    h.scm_solve(Bt, g_rhs, ld, ld, 1, stream)
    torch.cuda.synchronize()
    e_s0, e_s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_s0.record(stream)
    for _ in range(3):
        g_rhs.fill_(1.0)
        h.scm_solve(Bt, g_rhs, ld, ld, 1, stream)
    e_s1.record(stream)
    e_s1.synchronize()
    sce_ms = e_s0.elapsed_time(e_s1) / 3

    # end to end through the public host-buffer API (H2D inputs + D2H diag(R), info)
    rd = np.zeros(m)
    h.iteration_host(inst.xbar, inst.y, rd)
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(2, min(args.steps, 5))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        info = h.iteration_host(inst.xbar, inst.y, rd)
        e2e_t.append((time.perf_counter() - t0) * 1e3)
        assert info == 0
    e2e_ms = statistics.mean(e2e_t)

    if rank != 0:
        return None
    pk = peaks()
    ph = [statistics.mean(p[i] for p in phases) for i in range(8)]
    kt = [statistics.mean(p[i] for p in ktimes) for i in range(8)]
    upd_ms, n_upd, upd_flops = ph[5], ph[6], ph[7]
    fp64_derived = pk["bf16_sus"] * FP64_OVER_BF16
    achieved = upd_flops / (upd_ms * 1e-3) / 1e12 if upd_ms > 0 else None
    dmma = dfma = None
    if args.measure_peak:
        dmma, dfma = fp64_peak(local_rank, 1500.0)
    # roof = the larger of the derived FP64 figure and the DMMA throughput measured on this GPU
    fp64_peak_tf = max(fp64_derived, dmma or 0.0)
    peak_src = (f"builder-measured DMMA microbenchmark on this GPU ({dmma:.1f} TF/s, sdpc_fp64_peak; MEASURED_PEAKS "
                f"has no FP64 figure; > derived {fp64_derived:.1f} = {pk['src']} bf16 sustained {pk['bf16_sus']} x "
                f"nominal FP64/BF16 45/2250)"
                if dmma and dmma > fp64_derived else
                f"{pk['src']} bf16 sustained {pk['bf16_sus']} x FP64/BF16 nominal 45/2250")
    # per-phase roofline fractions (SURVEY §8(d) algorithmic work; kernel windows from CUDA events)
    trunc = inst.kind == "maxcut"
    fx, fy = solve_flops(st, inst, trunc)
    bbytes = 8.0 * entries(m)
    phase_roof = {
        "b_solve_x": {"flops": fx, "ms": kt[0], "tflops": fx / (kt[0] * 1e-3) / 1e12 if kt[0] > 0 else None},
        "b_solve_y": {"flops": fy, "ms": kt[1], "tflops": fy / (kt[1] * 1e-3) / 1e12 if kt[1] > 0 else None},
        "c_accumulate": {"bytes": bbytes, "ms": kt[2], "gbs": bbytes / (kt[2] * 1e-3) / 1e9 if kt[2] > 0 else None},
        "d_cholesky": {"flops": m ** 3 / 3.0, "ms": kt[3],
                       "tflops": m ** 3 / 3.0 / (kt[3] * 1e-3) / 1e12 if kt[3] > 0 else None},
        "note": ("(b): SURVEY 8(d) flops per RHS (etree-reach forward + backward over nnz(E[p:,p:]) when "
                 "max-cut truncation is on, + D scaling) over the solved RHS, per launch window (the X-hat "
                 "window overlaps (a2)); FP64 roof = the line's peak.  (c): B lower triangle written once "
                 "(8 m(m+1)/2 bytes) over the accumulate kernel; HBM roof = MEASURED_PEAKS hbm_gbs; "
                 "*_with_panel_reads adds the one read of the materialised truncated X-hat / Y^-1 panels the "
                 "unfused kernel needs (ncu: profiles/r02/final3/ncu_scm_trunc_full.txt, 0.84 GB read + 0.40 GB written).  (d): m^3/3 "
                 "over the Cholesky kernel."),
    }
    for key in ("b_solve_x", "b_solve_y", "d_cholesky"):
        v = phase_roof[key]["tflops"]
        phase_roof[key]["frac_fp64"] = v / fp64_peak_tf if v else None
    gbs = phase_roof["c_accumulate"]["gbs"]
    phase_roof["c_accumulate"]["frac_hbm"] = gbs / pk["hbm"] if gbs else None
    if inst.kind == "maxcut" and kt[2] > 0:
        # the unfused kernel also reads the materialised X-hat / Y^-1 panels once: rows i >= v of column v
        # (max-cut truncation), two arrays -> 2 * 8 * n(n+1)/2 bytes on top of the B write
        pbytes = bbytes + 2 * 8.0 * entries(inst.n)
        phase_roof["c_accumulate"]["bytes_with_panel_reads"] = pbytes
        phase_roof["c_accumulate"]["frac_hbm_with_panel_reads"] = pbytes / (kt[2] * 1e-3) / 1e9 / pk["hbm"]
    value = world * entries(m) / (ms * 1e-3)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "B-entries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "s_per_iter": ms * 1e-3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generator, instances/; SURVEY.md §8(d) recipe)",
        "config": {"workload": CONFIG_TEXT[args.config], "n": n, "m": m, "nnzE": int(inst.nnzE), "seed": args.seed,
                   "parallelism": "single GPU",
                   "l2": "256 MB buffer written between timed steps (L2 flush); step working set ~2.4 GB"},
        "phases_ms": {"start_to_a1_done": ph[0], "start_to_a2_done": ph[1], "start_to_b_done": ph[2],
                      "c_accumulate": ph[3], "d_cholesky": ph[4], "d_trailing_updates": upd_ms,
                      "note": "(a1) || (a2) on two streams, each factor's solves start when it is ready"},
        "clocks": clk.summary(),
        "next_rows": {"sce_solve_ms": sce_ms,
                      "note": "sdpc_scm_solve (R R^T) dz = g, one RHS, with the factor of the step (not in the metric)"},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "roofline": {"kernel": "chol_dag_kernel (SCM Cholesky (d): one persistent launch over the 128-tile task "
                               "graph, DMMA trailing updates)",
                     "bound": "tensor", "achieved": achieved, "peak": fp64_peak_tf, "unit": "TFLOP/s",
                     "frac": (achieved / fp64_peak_tf) if achieved else None,
                     "traffic": (DAG_BYTES_PER_FLOP * upd_flops) if DAG_BYTES_PER_FLOP else None,
                     "traffic_source": DAG_TRAFFIC_SOURCE,
                     "peak_source": peak_src,
                     "launches_per_step": n_upd, "flops_per_step": upd_flops,
                     "fp64_microbench_tflops": {"dmma": dmma, "dfma": dfma}},
        "phase_roofline": phase_roof,
        "e2e": {"value": world * entries(m) / (e2e_ms * 1e-3), "unit": "B-entries/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(2 * 8 * inst.nnzE),
                "d2h_bytes_per_step": int(8 * m + 4),
                "api": "sdpc_iteration_host (host xbar_E, y_E in; diag(R), info out)"},
    }
    if not args.no_cpu_baseline:
        cpu_baseline(inst, args)                 # warm-up (page cache, forked pool, BLAS init): not reported
        line["cpu_baseline"] = cpu_baseline(inst, args)
    return line


def run_ours_dist(args, rank, world, local_rank):
    """N > 1: one problem over N GPUs (strong scaling).  Each rank builds its 2D block-cyclic tiles of B
    (sdpc_scm_build with nranks = N) and the ranks factor B collectively inside the library
    (sdpc_scm_cholesky over the handle's NCCL communicators, created by sdpc_create from the 128-byte id
    of sdpc_get_unique_id that torch.distributed broadcasts).  SDPC_BENCH_BACKEND=gloo (test hook, ranks
    sharing one GPU) keeps the host-driven schedule of paper_1310_6919_b200/dist.py instead."""
    import numpy as np
    import torch

    import __graft_entry__
    from instances import gen_config

    __graft_entry__.build()
    from paper_1310_6919_b200 import Handle, dist as D
    from paper_1310_6919_b200.sdpc import get_unique_id

    dev = torch.device("cuda", local_rank)
    inst = gen_config(args.config, seed=args.seed)
    n, m = inst.n, inst.m
    dist = torch.distributed
    via_lib = os.environ.get("SDPC_BENCH_BACKEND", "nccl") == "nccl"
    uid = None
    if via_lib:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(get_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, src=0)
        uid = bytes(idt.cpu().numpy().tobytes())
    h = Handle.from_instance(inst, device=local_rank, nranks=world, rank=rank, nccl_id=uid)
    L = D.Layout(m, world, rank)
    lay = h.get_scm_layout()
    assert (lay["mloc"], lay["nloc"]) == (L.mloc, L.nloc)
    comm = None if via_lib else D.TorchComm(L)
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    Bt = torch.empty((max(1, L.nloc), L.lld), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step(timer=None, tb=None):
        h.factor_xinv(x, stream)
        h.scm_build(y, Bt, L.lld, stream)
        if tb is not None:
            tb.record(stream)
        if via_lib:
            info = h.scm_cholesky(Bt, L.lld, stream)
        else:
            info = D.dist_cholesky(h, Bt, L, comm, dev, stream, timer=timer)
        assert info == 0, info

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = h.launch_count()
    times, builds, upd = [], [], []
    ev0, evb, ev1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            timer = []
            step(timer, evb)
            ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            builds.append(ev0.elapsed_time(evb))
            upd.append((sum(a.elapsed_time(b) for a, b, _ in timer), sum(f for _, _, f in timer), len(timer)))
    launches = h.launch_count() - l0
    t = torch.tensor([statistics.mean(times), statistics.mean(builds)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, build_ms = float(t[0]), float(t[1])

    # end to end: pinned host inputs -> device every step, info back to the host
    xh = torch.from_numpy(inst.xbar).pin_memory()
    yh = torch.from_numpy(inst.y).pin_memory()
    e2e_t = []
    for _ in range(max(2, min(args.steps, 5))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        x.copy_(xh, non_blocking=True)
        y.copy_(yh, non_blocking=True)
        step()
        torch.cuda.synchronize()
        e2e_t.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([statistics.mean(e2e_t)], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te[0])
    if rank != 0:
        return None
    pk = peaks()
    from paper_1310_6919_b200 import fp64_peak
    dmma = fp64_peak(local_rank, 1500.0)[0] if args.measure_peak else None
    fp64_peak_tf = max(pk["bf16_sus"] * FP64_OVER_BF16, dmma or 0.0)
    if via_lib:
        # the whole distributed Cholesky (one library call per rank): m^3/3 over the max-rank time,
        # against world x the per-GPU FP64 roof
        upd_ms = ms - build_ms
        upd_fl = m ** 3 / 3.0
    else:
        upd_ms = statistics.mean(u[0] for u in upd)
        upd_fl = statistics.mean(u[1] for u in upd)
    achieved = upd_fl / (upd_ms * 1e-3) / 1e12 if upd_ms > 0 else None
    peak_all = fp64_peak_tf * (world if via_lib else 1)
    return {
        "metric": METRIC, "value": entries(m) / (ms * 1e-3), "unit": "B-entries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "s_per_iter": ms * 1e-3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, instances/; SURVEY.md §8(d) recipe)",
        "config": {"workload": CONFIG_TEXT[args.config], "n": n, "m": m, "nnzE": int(inst.nnzE), "seed": args.seed,
                   "parallelism": f"{L.Pr}x{L.Pc} 2D block-cyclic B (256 tiles), replicated (a1)/(a2)",
                   "l2": "256 MB buffer written between timed steps (L2 flush)"},
        "phases_ms": {"build_a1_a2_b_c_max_rank": build_ms, "cholesky_max_rank": ms - build_ms,
                      "rank0_update_kernels": upd_ms},
        "clocks": clk.summary(),
        "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
        "roofline": {"kernel": ("sdpc_scm_cholesky over NCCL (2D block-cyclic, all ranks; DMMA tile kernels)"
                                if via_lib else "gemm_nt_kernel<DIST> (rank 0 local trailing updates, DMMA)"),
                     "bound": "tensor", "achieved": achieved, "peak": peak_all, "unit": "TFLOP/s",
                     "frac": (achieved / peak_all) if achieved else None, "traffic": None,
                     "peak_source": (f"{world} x per-GPU FP64 roof {fp64_peak_tf:.1f} TF/s (builder-measured DMMA "
                                     f"microbenchmark when available, else {pk['src']} bf16 sustained x 45/2250)"),
                     "launches_per_step": upd[0][2] if upd else 1, "flops_per_step": upd_fl},
        "e2e": {"value": entries(m) / (e2e_ms * 1e-3), "unit": "B-entries/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(2 * 8 * inst.nnzE), "d2h_bytes_per_step": 4,
                "api": "per rank: pinned host xbar_E, y_E -> device, sdpc_factor_xinv + sdpc_scm_build + "
                       "sdpc_scm_cholesky (collective over NCCL), info to host"},
    }


# ----------------------------------------------------------------------------- oracle (reference arm)

_POOL_STATE = {}


def _pool_init():
    """Single-threaded workers: BLAS threads inside a worker would oversubscribe the cores."""
    try:
        from threadpoolctl import threadpool_limits
        _POOL_STATE["limits"] = threadpool_limits(1)
    except Exception:
        pass


def _pool_columns(cols):
    """Worker of the FCFS column pool: full SCM columns for a block of constraint indices."""
    from oracle import scm as SCM
    st = _POOL_STATE
    return cols, SCM.scm_columns(st["inst"], cols, st["solver"], prep=st["prep"])


def _fcfs_columns(inst, solver, prep, cols, procs, block=32):
    """Algorithm 2: the SCM columns in a first-come-first-served queue over `procs` worker
    processes (forked: the oracle's factors are shared copy-on-write), single-threaded solves inside a
    worker.  Returns B[:, cols] (m x len(cols)) and the wall time."""
    import multiprocessing as mp

    import numpy as np
    _POOL_STATE.update(inst=inst, solver=solver, prep=prep)
    blocks = [cols[a:a + block] for a in range(0, len(cols), block)]
    pos = {l: a for a, l in enumerate(cols)}
    out = np.zeros((inst.m, len(cols)))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs, initializer=_pool_init) as pool:
        for bc, val in pool.imap_unordered(_pool_columns, blocks):
            out[:, [pos[l] for l in bc]] = val
    return out, time.perf_counter() - t0


def cpu_baseline(inst, args, full=None):
    """The CPU oracle (oracle/, as it stands) timed for one iteration on this host's cores:
    Algorithm 1 (oracle), the Y factorisation, the SCM columns by sparse solves in an FCFS process pool
    (Algorithm 2), and LAPACK potrf at the true m.  Configs 0-2 build the full B (no extrapolation);
    larger configs time two column samples (1x and 3x) and fit t = t_fixed + t_col |cols|, scaling only
    t_col to m columns (labelled extrapolated)."""
    import numpy as np

    from oracle import algorithm1 as A1, cholesky as CH, scm as SCM, symbolic as SYM
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    t_sym = time.perf_counter() - t0
    t0 = time.perf_counter()
    L, D = A1.factor_xinv(S, inst.xbar)
    t_a1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    solver = SCM.ColumnSolver(S, L, D, inst.y, inst.perm)
    t_fac = time.perf_counter() - t0
    t0 = time.perf_counter()
    prep = SCM.column_prep(inst)
    t_prep = time.perf_counter() - t0
    m = inst.m
    if full is None:
        full = args.config in (0, 1, 2)
    if full:
        B, t_cols = _fcfs_columns(inst, solver, prep, list(range(m)), cores)
        t0 = time.perf_counter()
        CH.potrf_lower(B)
        t_chol = time.perf_counter() - t0
        t_build = t_prep + t_cols
        how = (f"full B ({m} columns) by the FCFS pool ({t_cols:.2f} s) + LAPACK potrf of that B, m = {m} "
               f"({t_chol:.2f} s)")
    else:
        rng = np.random.default_rng(1)
        n1 = max(2 * cores, 64)
        c1 = sorted(rng.choice(m, size=min(n1, m), replace=False).tolist())
        c3 = sorted(rng.choice(m, size=min(3 * n1, m), replace=False).tolist())
        _, ta = _fcfs_columns(inst, solver, prep, c1, cores)
        _, tb = _fcfs_columns(inst, solver, prep, c3, cores)
        t_col = max(tb - ta, 1e-9) / max(len(c3) - len(c1), 1)
        t_fixed = max(ta - t_col * len(c1), 0.0)
        t_build = t_prep + t_fixed + t_col * m
        # potrf at the true m if host memory allows (2 copies of m^2 doubles), else m^3-scaled from m/2
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        except (ValueError, OSError):
            avail = 0
        msub = m if 3 * 8 * m * m < avail else m // 2
        G = rng.standard_normal((msub, 64))
        Bs = G @ G.T / 64 + np.eye(msub)
        del G
        t0 = time.perf_counter()
        CH.potrf_lower(Bs)
        t_chol = (time.perf_counter() - t0) * (m / msub) ** 3
        del Bs
        how = (f"columns: two FCFS-pool samples ({len(c1)} cols {ta:.2f} s, {len(c3)} cols {tb:.2f} s) fitted "
               f"t = {t_fixed:.2f} s + {t_col * 1e3:.3f} ms x cols, EXTRAPOLATED to {m} columns; LAPACK potrf of "
               f"an SPD {msub}x{msub} ({'true m' if msub == m else 'm/2, x8: extrapolated'}, {t_chol:.2f} s)")
    t_iter = t_a1 + t_fac + t_build + t_chol
    return {"value": entries(m) / t_iter, "unit": "B-entries/s", "s_per_iter": t_iter, "cores": cores,
            "kind": "oracle",
            "phases_s": {"a1_algorithm1": t_a1, "y_factor": t_fac, "scm_columns": t_build, "potrf": t_chol},
            "sample": (f"oracle on {cores} host cores: Algorithm 1 on all cliques ({t_a1:.2f} s), Y factor ({t_fac:.2f} s), "
                       f"{how}; one-time symbolic setup {t_sym:.2f} s excluded")}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    from instances import gen_config
    inst = gen_config(args.config, seed=args.seed)
    vals = []
    # CPU steps have no caches to warm beyond the first: at most one warm-up step
    warm = min(args.warmup, 1)
    for i in range(warm + args.steps):
        cb = cpu_baseline(inst, args)
        if i >= warm:
            vals.append(cb)
    ms = statistics.mean(v["s_per_iter"] for v in vals) * 1e3
    value = entries(inst.m) / (ms * 1e-3)
    last = vals[-1]
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "B-entries/s", "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[args.config], "n": inst.n, "m": inst.m, "seed": args.seed},
            "steps_s": [v["s_per_iter"] for v in vals],
            "cpu_baseline": {"value": value, "unit": "B-entries/s", "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": "B-entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4, 5, 6])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--measure-peak", action="store_true", default=True)
    ap.add_argument("--no-measure-peak", dest="measure_peak", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (not used by the driver): run the N-rank schedule on fewer GPUs with gloo, e.g.
    # SDPC_BENCH_BACKEND=gloo SDPC_BENCH_DEVICE=0 torchrun --nproc-per-node 2 bench.py --gpus 2
    backend = os.environ.get("SDPC_BENCH_BACKEND", "nccl")
    if "SDPC_BENCH_DEVICE" in os.environ:
        local_rank = int(os.environ["SDPC_BENCH_DEVICE"])
    if world > 1 and args.impl == "ours":
        import torch
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group(backend)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and args.impl == "ours":
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
