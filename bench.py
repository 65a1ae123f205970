#!/usr/bin/env python
"""RSRS benchmark (BASELINE.json metric: factorization DOF/s excl. sampling + solve time).

One step = restore the four sample arrays from pristine device copies (the sweep
overwrites them in place) + rsrs_factor + rsrs_solve (1 RHS), i.e. one pass of the
whole hot path over one seeded synthetic problem.
value = DOF / step time (N points per step, summed over ranks), CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

Workload (default): c5 of BASELINE.json -- N = 1,048,576 Fibonacci-sphere points,
3D Laplace second-kind kernel, FP64, octree leaf 64, eps = 1e-6 -- the largest
configuration, and it fits one B200 (the 40.8 GB sample store twice: pristine +
working copy).  Inputs are far larger than L2 (no flush needed).  Sampling
(Y = A Omega, Z = A^* Psi through the harness kernel matvec) is done once before
timing (excluded, BASELINE.json north_star) and reported as sample_s.
N > 1 (torchrun): ONE problem sharded over the ranks (strong scaling): each rank
owns a Morton range of leaves, draws its own sample rows, and the sweep exchanges
near-field halo rows per colour and skeleton rows per level over NCCL
(include/rsrs.h multi-GPU section).

cpu_baseline / --impl reference: the CPU oracle (oracle/, test infrastructure) as it
stands, timed on this host's cores: a full factor + solve of the same configuration
family (kernel, p, eps, g, c_id, leaf) at a bounded N (default 8192 for the sphere),
its samples formed on the CPU from the dense operator (untimed), boxes of one colour
on nproc worker threads (one BLAS thread each).
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
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-n", type=int, default=0,
                    help="oracle sample size N (same config family); 0 = auto (sphere 8192, 2D grid 64x64)")
    ap.add_argument("--noise-factor", type=float, default=0.0,
                    help="f1: noise-aware tolerance atol(l-1) = max(atol(l), theta nu(l)) (0: fixed schedule)")
    ap.add_argument("--triangular", action="store_true",
                    help="f4: triangular (Cholesky) output form; needs --variant symmetric (spd operators)")
    ap.add_argument("--variant", default="paper", choices=["paper", "symmetric"],
                    help="paper: two independent sketches (PAPER.md:1180-1183, the headline); symmetric: the "
                         "SURVEY 8(f) f2 shortcut Psi = Omega, Z = Y for real symmetric A (c1-c3, c5) / "
                         "Psi = conj(Omega), Z = conj(Y) for the complex-symmetric c4")
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
    if symmetric:            # f2: Psi = Omega (real) / conj(Omega) (complex symmetric c4) => Z = Y / conj(Y);
        #                      only Y / Omega are read by the library
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
                 nranks=pb["world"], symmetric=pb["symmetric"], estimate_coupling=estimate and not pb["triangular"],
                 noise_factor=pb["noise_factor"], triangular=pb["triangular"])
    if solve_events is not None:
        solve_events[0].record(stream)
    f.solve(x, stream=stream)
    if solve_events is not None:
        solve_events[1].record(stream)
    return f


# ---------------------------------------------------------------------------
# CPU oracle baseline: a full factor + solve of a bounded member of the workload family
# ---------------------------------------------------------------------------
def oracle_config(cfg, n: int = 0):
    """Same kernel / p / eps / g / c_id / leaf as cfg at a bounded size."""
    if cfg.geometry == "grid2d":
        return cfg.scaled(n or 64)          # 64 x 64 grid (c1 size)
    return cfg.scaled(n or 8192)


def oracle_problem(cfg_s):
    """Dense operator and seeded samples of the bounded oracle case (CPU, untimed)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    import oracle as O
    import workloads as W
    X = W.points(cfg_s)
    t = O.build_tree(X, cfg_s.leaf, *cfg_s.root())
    with threadpool_limits(limits=os.cpu_count()):
        A = W.dense_matrix(cfg_s, X)
        Om, Ps = W.omega_psi(cfg_s)
        Y, Z = W.dense_samples(A, Om, Ps)
        P = t.perm
        arrays = [np.ascontiguousarray(M[P]) for M in (Y, Z, Om, Ps)]
    b = W.rhs(cfg_s)
    return dict(cfg=cfg_s, X=X, A=A, tree=t, arrays=arrays, b=b)


def oracle_run(pb, workers: int):
    """One timed oracle factor + solve (the oracle as it stands; inputs copied outside the timing)."""
    import numpy as np

    import oracle as O
    cfg_s = pb["cfg"]
    Yc, Zc, Oc, Pc = (M.copy() for M in pb["arrays"])
    t0 = time.perf_counter()
    f = O.factor(pb["tree"], Yc, Zc, Oc, Pc, cfg_s.eps, c_id=cfg_s.c_id, g=cfg_s.g, l=cfg_s.l, copy=False,
                 workers=workers)
    t1 = time.perf_counter()
    x = O.solve(f, pb["b"])
    t2 = time.perf_counter()
    res = float(np.linalg.norm(pb["A"] @ x - pb["b"]) / np.linalg.norm(pb["b"]))
    return t2 - t0, t1 - t0, t2 - t1, res


def host_desc():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = ""
    try:
        from threadpoolctl import threadpool_info
        for d in threadpool_info():
            if d.get("user_api") == "blas":
                blas = f"{d.get('internal_api')} {d.get('version')}"
                break
    except Exception:  # noqa: BLE001
        pass
    return model, blas


def oracle_baseline(cfg, n: int = 0, reps: int = 1, warm: int = 0):
    """cpu_baseline record: the oracle's full factor + solve of the bounded case, DOF/s."""
    pb = oracle_problem(oracle_config(cfg, n))
    workers = os.cpu_count() or 1
    times = [oracle_run(pb, workers) for _ in range(warm + reps)][warm:]
    tot = sum(t[0] for t in times)
    cfg_s = pb["cfg"]
    model, blas = host_desc()
    desc = (f"oracle factor + solve (every level, top block, 1-RHS solve) of {cfg_s.name}: {cfg.kernel}, "
            f"N = {cfg_s.N}, L = {pb['tree'].L}, p = {cfg_s.p}, eps = {cfg_s.eps}, g = {cfg_s.g}, c_id = {cfg_s.c_id}; "
            f"samples from the dense operator (untimed); {workers} worker threads x 1 BLAS thread ({blas}); "
            f"CPU: {model}")
    rec = {"value": cfg_s.N * len(times) / tot, "unit": "DOF/s", "cores": workers, "kind": "oracle",
           "sample": desc, "seconds_per_run": tot / len(times), "factor_s": times[-1][1], "solve_s": times[-1][2],
           "residual": times[-1][3], "N": cfg_s.N, "cpu_model": model, "blas": blas}
    return rec, times


# ---------------------------------------------------------------------------
def run_reference(args, rank, world, pg):
    import workloads as W
    if rank != 0:
        return
    cfg = W.CONFIGS[args.config]
    # every step is one full oracle factor + solve of a bounded member of the family, sized so the
    # whole --steps K --warmup W run stays within a few minutes (sphere: N = 4096, ~7 s per run on
    # 16 cores; 2D grid: 32 x 32); --cpu-n overrides
    n = args.cpu_n or (4096 if cfg.geometry == "sphere" else 32)
    rec, times = oracle_baseline(cfg, n, reps=args.steps, warm=args.warmup)
    tot = sum(t[0] for t in times)
    val = rec["value"]
    line = {"metric": METRIC, "value": val, "unit": "DOF/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "N": cfg.N, "p": cfg.p, "eps": cfg.eps,
                       "sample": rec["sample"], "same_config": False},
            "cpu_baseline": rec,
            "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_native(args, rank, world, local, pg):
    import numpy as np  # noqa: F401
    import torch

    import workloads as W
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    cfg = W.CONFIGS[args.config]
    if args.triangular and args.variant != "symmetric":
        raise SystemExit("--triangular needs --variant symmetric (the triangular form is for spd operators)")
    pb = setup_problem(cfg, dev, rank, world, pg, symmetric=args.variant == "symmetric")
    pb["noise_factor"] = args.noise_factor
    pb["triangular"] = args.triangular
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
    atols = {str(lev): f.atol(lev) for lev in range(st["L"], st["top_level"] - 1, -1)}
    if world == 1 and not pb["triangular"]:
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
                                      "atol": fe.atol(lev)}
        del fe
    # ---- e2e: the same step through the C ABI with PINNED HOST buffers: rsrs_factor reads the host
    # samples (Omega / Psi copied up front, the Y / Z rows of each leaf colour batch streamed one batch
    # ahead of the sweep), rsrs_solve takes the host right-hand side; every H2D / D2H byte is inside
    # the timed region.  World > 1 keeps device inputs plus explicit copies (host mode is single-rank).
    e2e = None
    if not args.no_e2e:
        def pinned_copy(t):        # pinned host buffer filled from the device (no pageable staging copy)
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h
        host = [pinned_copy(t) for t in pb["src"]]
        hb = pinned_copy(pb["b"])
        hx = torch.empty(hb.shape, dtype=hb.dtype, pin_memory=True)
        h2d = sum(t.numel() * t.element_size() for t in host) + hb.numel() * hb.element_size()
        d2h = hx.numel() * hx.element_size()
        del work[:]
        f = None
        torch.cuda.empty_cache()
        import paper_2311_01451_b200 as R
        R.release_memory()          # idle arena chunks back to the driver (host mode owns a device store)
        barrier(pg, dev)
        torch.cuda.synchronize(dev)
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.e2e_steps):
            if world == 1:
                hx.copy_(hb)
                f = None
                f = factor_solve(pb, host, hx, stream)
            else:
                wk = [torch.empty_like(t) for t in pb["src"]]
                with torch.cuda.stream(stream):
                    for w, h in zip(wk, host):
                        w.copy_(h, non_blocking=True)
                    x.copy_(hb, non_blocking=True)
                f = None
                f = factor_solve(pb, wk, x, stream)
                with torch.cuda.stream(stream):
                    hx.copy_(x, non_blocking=True)
                del wk
        g1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(pg, dev)
        gms = max_over_ranks(g0.elapsed_time(g1), pg, dev)
        e2e = {"value": N * args.e2e_steps / (gms * 1e-3), "unit": "DOF/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": gms / args.e2e_steps,
               "path": "rsrs_factor / rsrs_solve on pinned host buffers (library-side overlapped transfer)"
               if world == 1 else "explicit H2D copies + device rsrs_factor"}
    if rank != 0:
        return
    # ---- roofline of the dominant kernel (live CUDA-event times inside the timed region)
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    name, d = dom
    per_launch_ms = d["ms"] / max(d["launches"], 1)
    achieved = d["flops"] / (d["ms"] * 1e-3) / 1e12
    peak = peaks.get("dmma_tflops")
    # DRAM bytes per class region (one NVTX range = one colour batch's launches of the class),
    # dram__bytes_read.sum + dram__bytes_write.sum from an ncu capture of THIS config
    # (tools/ncu_traffic.py -> profiles/ncu_traffic_r02.json); None if not captured.
    traffic, traffic_src = None, None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
    if os.path.exists(tfile):
        try:
            rec = json.load(open(tfile)).get(cfg.name, {}).get(name)
            if rec:
                traffic, traffic_src = rec["bytes_per_region"], rec.get("source")
        except Exception:  # noqa: BLE001
            traffic = None
    nreg = max(d["launches"], 1)
    roof = {"bound": "tensor", "kernel": name, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if peak else None, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": "measured FP64 DMMA (tools/fp64_peak, this box; MEASURED_PEAKS.json has no FP64)",
            "launch_unit": "one class region = the launches of the class for one colour batch (an NVTX range)",
            "flops_per_launch": d["flops"] / nreg, "bytes_model_per_launch": d["bytes"] / nreg,
            "ms_per_launch": per_launch_ms, "launches": d["launches"] // max(args.steps, 1),
            "share_of_step": d["ms"] / ms}
    breakdown = {k: {"ms_per_step": v["ms"] / args.steps, "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9,
                     "gbs": v["bytes"] / max(v["ms"], 1e-9) / 1e6} for k, v in prof.items() if v["launches"]}
    cpu = None
    if not args.no_cpu and world == 1:
        cpu, _ = oracle_baseline(cfg, args.cpu_n, reps=1)
    sweep_tf = st["flops_model"] / (st["factor_ms"] * 1e-3) / 1e12
    sweep_tf_s = st["flops_survey"] / (st["factor_ms"] * 1e-3) / 1e12
    sweep = {"build_model_tflop": st["flops_model"] / 1e12, "build_model_tflops": sweep_tf,
             "survey_model_tflop": st["flops_survey"] / 1e12, "survey_model_tflops": sweep_tf_s,
             "survey_model_frac": (sweep_tf_s / peak) if peak else None,
             "note": "whole factor sweep: build model = this build's formulation (CholeskyQR, Gram blocks); "
                     "survey model = SURVEY 8(d) standard dense forms on the same (n_b, r, k)"}
    line = {"metric": METRIC, "value": N * args.steps / (ms * 1e-3), "unit": "DOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "N": N, "p": cfg.p, "eps": cfg.eps, "g": cfg.g, "leaf": cfg.leaf,
                       "kernel": cfg.kernel, "L": st["L"], "l2": f"inputs {sum(t.numel() * t.element_size() for t in pb['src']) / 1e9:.1f} GB > 126 MB L2 (no flush needed)",
                       "step": "restore samples + rsrs_factor + rsrs_solve(1 rhs)", "variant": args.variant + (f", noise-aware tolerance theta = {args.noise_factor}" if args.noise_factor else "")
                       + (", triangular form" if args.triangular else ""), "parallelism": (f"morton-range x{world}, halo exchange, gather at level {pb['gather_level']}"
                                       if world > 1 else "single GPU")},
            "factor_ms": st["factor_ms"], "solve_ms": statistics.median(solve_ms), "sample_s": pb["t_sample"], "tree_s": pb["t_tree"],
            "residual": resid, "top_size": st["top_size"], "max_rank": st["max_rank"],
            "memory_scalars": st["memory_scalars"], "sweep": sweep,
            "roofline": roof, "kernels": breakdown, "fp64_peaks": peaks, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk, "coupling_estimate": coupling, "atol_per_level": atols}
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
