#!/usr/bin/env python
"""RSRS benchmark (BASELINE.json metric: factorization DOF/s excl. sampling + solve time).

One step = restore the four sample arrays from pristine device copies (the sweep
overwrites them in place) + rsrs_factor + rsrs_solve (1 RHS), i.e. one pass of the
whole hot path over one seeded synthetic problem.
value = DOF / step time (N points per step, summed over ranks), CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

Workload: configs[1] of BASELINE.json (c2: 512 x 512 grid, 2D log kernel, FP64,
N = 262144, eps = 1e-6) -- inputs (Y, Z, Omega, Psi: 6.4 GB) are larger than L2, so
no explicit L2 flush is needed.  Sampling (Y = A Omega, Z = A^* Psi through the
harness kernel matvec) is done once before timing (excluded, BASELINE.json
north_star).  N > 1 (torchrun): ONE problem sharded over the ranks (strong scaling): each rank
owns a Morton range of leaves, draws its own sample rows, and the sweep exchanges
near-field halo rows per colour and skeleton rows per level over NCCL
(include/rsrs.h multi-GPU section); the solve takes the
replicated right-hand side.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RSRS factorization DOF/s (excl. sampling) + solve time; FP64 FLOP/s & HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-boxes", type=int, default=0, help="oracle sample size (leaf boxes); 0 = auto")
    ap.add_argument("--variant", default="paper", choices=["paper", "symmetric"],
                    help="paper: two independent sketches (PAPER.md:1180-1183, the headline); symmetric: the "
                         "SURVEY 8(f) f2 shortcut Psi = Omega, Z = Y for real symmetric A")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (torchrun); one process per GPU
# ---------------------------------------------------------------------------
def dist_init(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "native" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        pg = dist
    return rank, world, local, pg


def max_over_ranks(x: float, pg, device=None) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg, device=None):
    if pg is not None:
        if device is not None:
            pg.barrier(device_ids=[device.index])
        else:
            pg.barrier()


# ---------------------------------------------------------------------------
# clocks during the timed region (nvidia-smi sampler)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak() -> dict:
    """Measured FP64 peaks (tools/fp64_peak: DMMA and DFMA loops); MEASURED_PEAKS.json has none."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout.strip().splitlines()[-1]
        return json.loads(out)
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


# ---------------------------------------------------------------------------
# problem setup (seeded, synthetic; sampling excluded from timing)
# ---------------------------------------------------------------------------
def setup_problem(cfg, dev, rank=0, world=1, pg=None, symmetric=False):
    """Seeded problem; with world > 1 this rank keeps only its Morton range of rows
    (rsrs_tree_partition) and draws its own sample rows Y = A[rows, :] Omega."""
    import numpy as np
    import torch

    import paper_2311_01451_b200 as R
    import workloads as W
    X = W.points(cfg)
    t_tree = time.perf_counter()
    tree = R.Tree(X, cfg.leaf, *cfg.root(), nranks=world)
    t_tree = time.perf_counter() - t_tree
    perm = tree.perm()
    N = cfg.N
    first, gather = tree.partition(world)
    r0, r1 = int(first[rank]), int(first[rank + 1])
    Om, Ps = W.omega_psi(cfg)
    P = torch.from_numpy(perm).to(dev)
    Om_d = torch.from_numpy(Om).to(dev)[P].contiguous()
    Ps_d = torch.from_numpy(Ps).to(dev)[P].contiguous()
    del Om, Ps
    pts = np.zeros((N, 3))
    pts[:, :X.shape[1]] = X
    pts_d = torch.from_numpy(pts[perm]).to(dev)
    Y_d = torch.empty((r1 - r0, cfg.p), dtype=Om_d.dtype, device=dev)
    Z_d = torch.empty_like(Y_d)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    R.sample_matvec_rows(cfg.kernel, pts_d, W.kernel_weight(cfg), Om_d, Y_d, r0, kappa=cfg.kappa)
    if symmetric:            # f2: Psi = Omega => Z = A^T Omega = Y; only Y / Omega are used
        Ps_d, Z_d = Om_d, Y_d
    else:
        R.sample_matvec_rows(cfg.kernel, pts_d, W.kernel_weight(cfg), Ps_d, Z_d, r0, adjoint=True,
                             kappa=cfg.kappa)
    torch.cuda.synchronize(dev)
    t_sample = time.perf_counter() - t0
    if world > 1:
        Om_d = Om_d[r0:r1].contiguous()
        Ps_d = Ps_d[r0:r1].contiguous()
        torch.cuda.empty_cache()
    b = torch.from_numpy(W.rhs(cfg)).to(dev)
    comm = None
    if world > 1:
        def bcast(raw):
            obj = [raw]
            pg.broadcast_object_list(obj, src=0)
            return obj[0]
        comm = R.NcclComm(world, rank, bcast)
    src = [Y_d, Om_d] if symmetric else [Y_d, Z_d, Om_d, Ps_d]
    return dict(cfg=cfg, X=X, tree=tree, perm=perm, P=P, pts=pts_d, src=src, b=b, symmetric=symmetric,
                t_sample=t_sample, t_tree=t_tree, comm=comm, rank=rank, world=world, rows=(r0, r1),
                gather_level=gather)


def factor_solve(pb, work, x, stream, profile=False, solve_events=None, estimate=False):
    import paper_2311_01451_b200 as R
    cfg = pb["cfg"]
    arrays = (work[0], None, work[1], None) if pb["symmetric"] else tuple(work)
    f = R.factor(pb["tree"], *arrays, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
                 oversample=cfg.l, stream=stream, profile=profile, comm=pb["comm"], rank=pb["rank"],
                 nranks=pb["world"], symmetric=pb["symmetric"], estimate_coupling=estimate)
    if solve_events is not None:
        solve_events[0].record(stream)
    f.solve(x, stream=stream)
    if solve_events is not None:
        solve_events[1].record(stream)
    return f


# ---------------------------------------------------------------------------
# CPU oracle baseline on a bounded sample (leaf boxes of the same workload)
# ---------------------------------------------------------------------------
def oracle_sample(cfg, nboxes: int, reps: int = 1, seed_offset: int = 0):
    """Time the oracle on the first `nboxes` leaf boxes of the canonical order.

    Those boxes (colour 0 of the leaf level) read only their own Y/Z rows and the
    near-field Omega/Psi rows, so their samples are computed exactly on the CPU by
    direct sums (no GPU involvement) and the oracle's per-box work is the full
    O4-O9 sequence of the workload.  Returns DOF/s = (points eliminated or
    skeletonised in the sample) / time, plus the sample description.
    """
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle as O
    import workloads as W
    X = W.points(cfg)
    t = O.build_tree(X, cfg.leaf, *cfg.root())
    N, p, L = cfg.N, cfg.p, t.L
    lv = t.levels[L]
    order = t.canonical_order(L)[:nboxes]
    Om, Ps = W.omega_psi(cfg)
    Om, Ps = Om[t.perm], Ps[t.perm]
    Y = np.zeros_like(Om)
    Z = np.zeros_like(Ps)
    allidx = np.arange(N)
    with threadpool_limits(limits=os.cpu_count()):
        for b in order:
            rows = np.arange(lv.start[b], lv.start[b + 1])
            Ab = W.kernel_block(cfg, X, t.perm[rows], t.perm[allidx])
            Y[rows] = Ab @ Om
            Z[rows] = Ab.conj() @ Ps        # A^* rows = conj(A)^T rows (symmetric kernels)
    times = []
    dofs = int(sum(lv.start[b + 1] - lv.start[b] for b in order))
    with threadpool_limits(limits=1):
        for _ in range(reps):
            Yc, Zc, Oc, Pc = Y.copy(), Z.copy(), Om.copy(), Ps.copy()
            t0 = time.perf_counter()
            O.factor(t, Yc, Zc, Oc, Pc, cfg.eps, c_id=cfg.c_id, g=cfg.g, l=cfg.l, max_boxes=len(order), copy=False)
            times.append(time.perf_counter() - t0)
    return dofs, times, f"oracle O4-O9 on the first {len(order)} leaf boxes (colour 0, {dofs} points) of {cfg.name}"


# ---------------------------------------------------------------------------
def run_reference(args, rank, world, pg):
    import workloads as W
    if rank != 0:
        return
    cfg = W.CONFIGS[args.config]
    nb = args.cpu_boxes or 24
    dofs, times, desc = oracle_sample(cfg, nb, reps=args.warmup + args.steps)
    timed = times[args.warmup:]
    tot = sum(timed)
    val = dofs * len(timed) / tot
    line = {"metric": METRIC, "value": val, "unit": "DOF/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(timed), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "N": cfg.N, "p": cfg.p, "eps": cfg.eps, "sample": desc},
            "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_native(args, rank, world, local, pg):
    import numpy as np  # noqa: F401
    import torch

    import workloads as W
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    cfg = W.CONFIGS[args.config]
    if args.variant == "symmetric" and cfg.is_complex:
        raise SystemExit("--variant symmetric needs a real symmetric operator (not c4)")
    pb = setup_problem(cfg, dev, rank, world, pg, symmetric=args.variant == "symmetric")
    stream = torch.cuda.Stream(device=dev)
    work = [t.clone() for t in pb["src"]]
    x = pb["b"].clone()
    N = cfg.N
    peaks = fp64_peak() if rank == 0 else {}

    def step(profile=False, solve_events=None):
        with torch.cuda.stream(stream):
            for w, s in zip(work, pb["src"]):
                w.copy_(s)
            x.copy_(pb["b"])
        return factor_solve(pb, work, x, stream, profile=profile, solve_events=solve_events)

    f = None
    for _ in range(args.warmup):
        f = None
        f = step()
    torch.cuda.synchronize(dev)
    # ---- timed region -------------------------------------------------------
    clocks = Clocks(local)
    prof = {}
    launches = 0
    barrier(pg, dev)
    torch.cuda.synchronize(dev)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    solve_ms = []
    for _ in range(args.steps):
        f = None
        sev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        f = step(profile=True, solve_events=sev)
        sev[1].synchronize()
        solve_ms.append(sev[0].elapsed_time(sev[1]))
        for c in f.profile():
            a = prof.setdefault(c["name"], {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
            a["ms"] += c["ms"]
            a["flops"] += c["flops"]
            a["bytes"] += c["bytes"]
            a["launches"] += c["launches"]
        st = f.stats()
        launches += st["launches"] + st["solve_launches"]
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier(pg, dev)
    ms_local = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms = max_over_ranks(ms_local, pg, dev)
    st = f.stats()
    # residual of the last solve via the harness operator (property that holds at any size)
    import paper_2311_01451_b200 as R
    ax = torch.empty_like(x)
    xt = x[pb["P"]].contiguous()
    R.sample_matvec(cfg.kernel, pb["pts"], W.kernel_weight(cfg), xt.view(N, 1), ax.view(N, 1), kappa=cfg.kappa)
    resid = float((ax - pb["b"][pb["P"]]).norm() / pb["b"].norm())
    # ---- coupling estimates, one extra factorization outside the timed region
    coupling = None
    if world == 1:
        with torch.cuda.stream(stream):
            for w_, s_ in zip(work, pb["src"]):
                w_.copy_(s_)
            x.copy_(pb["b"])
        fe = factor_solve(pb, work, x, stream, estimate=True)
        coupling = {}
        tr = pb["tree"]
        for lev in range(st["L"], st["top_level"] - 1, -1):
            nbx = len(tr.level(lev)["keys"])
            e = fe.coupling(lev, nbx)
            e = e[e[:, 0] >= 0]
            if e.size:
                coupling[str(lev)] = {"max": float(e.max()), "median": float(np.median(e)),
                                      "atol": cfg.c_id * cfg.eps * cfg.g ** (st["L"] - lev)}
        del fe
    # ---- e2e: host (pinned) inputs, H2D + factor + solve + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in pb["src"]]
        hb = pb["b"].cpu().pin_memory()
        hx = torch.empty_like(hb).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in host) + hb.numel() * hb.element_size()
        d2h = hx.numel() * hx.element_size()
        barrier(pg, dev)
        torch.cuda.synchronize(dev)
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.e2e_steps):
            with torch.cuda.stream(stream):
                for w, h in zip(work, host):
                    w.copy_(h, non_blocking=True)
                x.copy_(hb, non_blocking=True)
            f = None
            f = factor_solve(pb, work, x, stream)
            with torch.cuda.stream(stream):
                hx.copy_(x, non_blocking=True)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(pg, dev)
        gms = max_over_ranks(g0.elapsed_time(g1), pg, dev)
        e2e = {"value": N * args.e2e_steps / (gms * 1e-3), "unit": "DOF/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": gms / args.e2e_steps}
    if rank != 0:
        return
    # ---- roofline of the dominant kernel (live CUDA-event times inside the timed region)
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    name, d = dom
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    achieved = d["flops"] / (d["ms"] * 1e-3) / 1e12
    peak = peaks.get("dmma_tflops")
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(name)
        except Exception:  # noqa: BLE001
            traffic = None
    roof = {"bound": "tensor", "kernel": name, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if peak else None, "traffic": traffic,
            "peak_source": "measured FP64 DMMA (tools/fp64_peak, this box; MEASURED_PEAKS.json has no FP64)",
            "flops_per_launch": d["flops"] / max(d["launches"], 1), "ms_per_launch": per_launch_ms,
            "share_of_step": d["ms"] / ms}
    breakdown = {k: {"ms_per_step": v["ms"] / args.steps, "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9,
                     "gbs": v["bytes"] / max(v["ms"], 1e-9) / 1e6} for k, v in prof.items() if v["launches"]}
    cpu = None
    if not args.no_cpu and world == 1:
        nbx = args.cpu_boxes or 96
        dofs, times, desc = oracle_sample(cfg, nbx, reps=1)
        cpu = {"value": dofs / times[0], "unit": "DOF/s", "cores": 1, "kind": "oracle", "sample": desc,
               "seconds": times[0]}
    sweep_tf = st["flops_model"] / (st["factor_ms"] * 1e-3) / 1e12
    line = {"metric": METRIC, "value": N * args.steps / (ms * 1e-3), "unit": "DOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "N": N, "p": cfg.p, "eps": cfg.eps, "g": cfg.g, "leaf": cfg.leaf,
                       "kernel": cfg.kernel, "L": st["L"], "l2": f"inputs {sum(t.numel() * t.element_size() for t in pb['src']) / 1e9:.1f} GB > 126 MB L2 (no flush needed)",
                       "step": "restore samples + rsrs_factor + rsrs_solve(1 rhs)", "variant": args.variant, "parallelism": (f"morton-range x{world}, halo exchange, gather at level {pb['gather_level']}"
                                       if world > 1 else "single GPU")},
            "factor_ms": st["factor_ms"], "solve_ms": statistics.median(solve_ms), "sample_s": pb["t_sample"], "tree_s": pb["t_tree"],
            "residual": resid, "top_size": st["top_size"], "max_rank": st["max_rank"],
            "memory_scalars": st["memory_scalars"], "sweep_tflops": sweep_tf,
            "roofline": roof, "kernels": breakdown, "fp64_peaks": peaks, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk, "coupling_estimate": coupling}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local, pg = dist_init(args)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world, pg)
        else:
            run_native(args, rank, world, local, pg)
    finally:
        if pg is not None:
            pg.destroy_process_group()


if __name__ == "__main__":
    main()
