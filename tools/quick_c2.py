"""Development tool: c2-scale sweep over (p, g) with one sampling at p_max."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_01451_b200 as R, workloads as W

name = os.environ.get("CFG", "c2")
cfg = W.CONFIGS[name]
if os.environ.get("NSIDE"):
    cfg = cfg.scaled(int(os.environ["NSIDE"]))
if os.environ.get("EPS"):
    from dataclasses import replace
    cfg = replace(cfg, eps=float(os.environ["EPS"]))
runs = [tuple(float(v) for v in x.split(":")) for x in os.environ.get("RUNS", "1024:1").split(",")]
pmax = max(int(r[0]) for r in runs)
ITERS = int(os.environ.get("ITERS", "2"))
dev = torch.device("cuda:0")
X = W.points(cfg)
t = R.Tree(X, cfg.leaf, *cfg.root())
perm = t.perm()
N = cfg.N
Om, Ps = W.omega_psi(cfg, p=pmax)
P = torch.from_numpy(perm).to(dev)
Om_d = torch.from_numpy(Om).to(dev)[P].contiguous(); Ps_d = torch.from_numpy(Ps).to(dev)[P].contiguous()
del Om, Ps
pts = np.zeros((N, 3)); pts[:, :X.shape[1]] = X
pts_d = torch.from_numpy(pts[perm]).to(dev)
Y_d = torch.empty_like(Om_d); Z_d = torch.empty_like(Ps_d)
torch.cuda.synchronize(); t0 = time.time()
R.sample_matvec(cfg.kernel, pts_d, W.kernel_weight(cfg), Om_d, Y_d, kappa=cfg.kappa)
R.sample_matvec(cfg.kernel, pts_d, W.kernel_weight(cfg), Ps_d, Z_d, adjoint=True, kappa=cfg.kappa)
torch.cuda.synchronize(); print("sample", time.time() - t0, flush=True)
src = [Y_d, Z_d, Om_d, Ps_d]
work = [x.clone() for x in src]
b = torch.from_numpy(W.rhs(cfg)).to(dev)
for (pf, g) in runs:
    p = int(pf)
    for it in range(ITERS):
        for w_, s_ in zip(work, src): w_.copy_(s_)
        torch.cuda.synchronize(); t0 = time.time()
        try:
            prof = os.environ.get("PROF", "last")
            f = R.factor(t, *work, p=p, eps=cfg.eps, level_growth=g, id_scale=cfg.c_id, oversample=cfg.l,
                         profile=(prof == "all" or (prof == "last" and it == ITERS - 1)))
        except R.RSRSError as e:
            print(f"p={p} g={g}: {e}", flush=True); break
        torch.cuda.synchronize(); t1 = time.time()
        x = b.clone(); f.solve(x); torch.cuda.synchronize(); t2 = time.time()
        st = f.stats()
        print(f"p={p} g={g} iter {it}: factor {1e3*(t1-t0):.1f} ms (dev {st['factor_ms']:.1f}), solve {1e3*(t2-t1):.2f} ms, "
              f"DOF/s {N/(t1-t0):.3e}, model {st['flops_model']/1e12:.2f} TF, {st['flops_model']/(st['factor_ms']*1e-3)/1e12:.2f} TF/s", flush=True)
    else:
        ax = torch.empty_like(x)
        R.sample_matvec(cfg.kernel, pts_d, W.kernel_weight(cfg), x[P].contiguous().view(N, 1), ax.view(N, 1), kappa=cfg.kappa)
        res = (ax - b[P]).norm() / b.norm()
        ks = []
        for lev in range(t.L, 1, -1):
            k = f.ranks(lev, len(t.level(lev)["keys"])); k = k[k >= 0]
            if k.size:
                ks.append(f"L{lev}:{k.min()}/{k.mean():.1f}/{k.max()}")
        print(f"p={p} g={g}: residual {res.item():.3e} |S| {st['top_size']} ranks {' '.join(ks)}", flush=True)
        for c in f.profile():
            if c["launches"]:
                print(f"   {c['name']:18s} {c['ms']:8.2f} ms  {c['flops']/1e9:9.1f} GF  {c['flops']/max(c['ms'],1e-9)/1e9:7.2f} TF/s  {c['bytes']/max(c['ms'],1e-9)/1e6:7.1f} GB/s  n={c['launches']}", flush=True)
