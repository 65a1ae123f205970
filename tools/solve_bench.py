"""Solve / apply timing: one factorization, then the median of 20 solves
with 1 and 16 right-hand sides (CUDA events on the launching stream), against the factor bytes M.
Harness tool (no oracle):  CFG=c2 python tools/solve_bench.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_01451_b200 as R  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[os.environ.get("CFG", "c2")]
dev = torch.device("cuda:0")
X = W.points(cfg)
t = R.Tree(X, cfg.leaf, *cfg.root())
perm = t.perm()
Om, Ps = W.omega_psi(cfg)
P = torch.from_numpy(perm).to(dev)
Om_d = torch.from_numpy(Om).to(dev)[P].contiguous()
Ps_d = torch.from_numpy(Ps).to(dev)[P].contiguous()
del Om, Ps
pts = np.zeros((cfg.N, 3))
pts[:, :X.shape[1]] = X
pts_d = torch.from_numpy(pts[perm]).to(dev)
Y_d = torch.empty_like(Om_d)
Z_d = torch.empty_like(Ps_d)
R.sample_matvec(cfg.kernel, pts_d, W.kernel_weight(cfg), Om_d, Y_d, kappa=cfg.kappa)
R.sample_matvec(cfg.kernel, pts_d, W.kernel_weight(cfg), Ps_d, Z_d, adjoint=True, kappa=cfg.kappa)
f = R.factor(t, Y_d, Z_d, Om_d, Ps_d, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id,
             oversample=cfg.l)
del Y_d, Z_d, Om_d, Ps_d
st = f.stats()
esz = 16 if cfg.is_complex else 8
M_bytes = st["memory_scalars"] * esz
s = torch.cuda.Stream()
out = {"config": cfg.name, "N": cfg.N, "factor_bytes": M_bytes, "launches_per_solve": st["solve_launches"]}
for nrhs in (1, 4, 16):
    B = torch.from_numpy(W.gaussian((cfg.N, nrhs), 3, 2, cfg.is_complex)).to(dev)
    if nrhs == 1:
        B = B[:, 0].contiguous()
    for what in ("solve", "apply"):
        ms = []
        for it in range(23):
            x = B.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            (f.solve if what == "solve" else f.apply)(x, stream=s)
            e1.record(s)
            e1.synchronize()
            if it >= 3:
                ms.append(e0.elapsed_time(e1))
        m = statistics.median(ms)
        out[f"{what}_{nrhs}rhs_ms"] = m
        out[f"{what}_{nrhs}rhs_GBs_on_M"] = M_bytes / (m * 1e-3) / 1e9
print(json.dumps(out))
