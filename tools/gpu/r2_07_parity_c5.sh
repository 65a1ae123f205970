#!/bin/bash
# round 2, call 7: full-size oracle parity on c5 (N = 1,048,576: ~45 min of oracle time on the host),
# then compute-sanitizer racecheck / synccheck of one c1 factorization + solve
mkdir -p gpurun_out
# Gram assembly A/B (per slot vs per box) on c3 first
for a in slot box; do
  RSRS_ASSEMBLE=$a CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_assemble_$a.log 2>&1
done
python tests/parity_full.py --config c5 --out gpurun_out/r02_parity_c5.json > gpurun_out/r2_parity_c5.log 2>&1
echo "c5 parity exit $?" > gpurun_out/r2_call7.txt
cat > /tmp/c1_once.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_01451_b200 as R, workloads as W
cfg = W.CONFIGS["c1"]
X = W.points(cfg); A = W.dense_matrix(cfg, X); Om, Ps = W.omega_psi(cfg); Y, Z = W.dense_samples(A, Om, Ps)
t = R.Tree(X, cfg.leaf, *cfg.root()); perm = t.perm()
T = [torch.from_numpy(np.ascontiguousarray(M[perm])).cuda() for M in (Y, Z, Om, Ps)]
f = R.factor(t, *T, p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id, oversample=cfg.l)
x = torch.from_numpy(W.rhs(cfg)).cuda(); f.solve(x); f.apply(x); torch.cuda.synchronize()
print("c1 once ok", f.stats()["launches"])
PY
for tool in racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/c1_once.py > gpurun_out/r2_sanitizer_$tool.log 2>&1
  echo "sanitizer $tool exit $?" >> gpurun_out/r2_call7.txt
done
