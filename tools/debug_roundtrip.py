import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import workloads as W, oracle as O
from gpu_common import dense_problem, run_gpu, run_oracle
cfg = W.CONFIGS["c1"]
X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
t_g, f_g = run_gpu(cfg, X, Y, Z, Om, Ps, cfg.root())
N = cfg.N
I = torch.eye(N, dtype=torch.float64, device="cuda:0")
K = I.clone(); f_g.apply(K)        # rows = original index i, col j: K e_j ... row-major N x N: B[:, j] is RHS j
Ki = I.clone(); f_g.solve(Ki)
K = K.cpu().numpy(); Ki = Ki.cpu().numpy()
E = Ki @ K - np.eye(N)
print("||Kinv K - I||", np.abs(E).max())
perm = t_g.perm(); inv = np.empty(N, int); inv[perm] = np.arange(N)
Et = E[np.ix_(perm, perm)]   # tree order
bad_rows = np.where(np.abs(Et).max(1) > 1e-9)[0]
bad_cols = np.where(np.abs(Et).max(0) > 1e-9)[0]
print("bad rows (tree pos)", len(bad_rows), bad_rows[:40])
print("bad cols (tree pos)", len(bad_cols), bad_cols[:40])
S = f_g.top()
print("|S|", len(S), "bad rows in S", np.isin(bad_rows, S).sum(), "bad cols in S", np.isin(bad_cols, S).sum())
print("K vs A", np.abs(K - A).max(), " Kinv vs inv(A)", np.abs(Ki - np.linalg.inv(A)).max())
# per-level eliminated sets from the oracle for reference
