#!/usr/bin/env python
"""DRAM traffic per kernel-class region for bench.py's roofline `traffic` field.

Every kernel-class region of rsrs_factor is an NVTX push/pop range named after the
class (factor.cu Planner::tic/toc), so ncu can attribute its launches:

  # 1. one factorization of the config under ncu, kernels renamed by their class range
  ncu --nvtx --nvtx-include "gemm_nt_gram/" --nvtx-include "gemm_nn_lu_update/" \
      --print-nvtx-rename kernel --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file gpurun_out/ncu_traffic_c5.csv \
      python tools/ncu_traffic.py run --config c5 --regions gpurun_out/regions_c5.json
  # 2. sum per class / number of class regions -> profiles/ncu_traffic_r02.json
  python tools/ncu_traffic.py parse --config c5 --csv gpurun_out/ncu_traffic_c5.csv \
      --regions gpurun_out/regions_c5.json --out profiles/ncu_traffic_r02.json

A region = all launches of the class for one colour batch (the unit bench.py's
`flops_per_launch` uses).  Harness only (no oracle, no timing claims).
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg_name: str, regions_out: str):
    import numpy as np
    import torch

    import paper_2311_01451_b200 as R
    import workloads as W
    cfg = W.CONFIGS[cfg_name]
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
    regions = {c["name"]: c["launches"] for c in f.profile()}
    with open(regions_out, "w") as fh:
        json.dump({"config": cfg_name, "regions": regions, "stats": f.stats()}, fh)


def parse(cfg_name: str, csv_path: str, regions_path: str, out: str):
    regions = json.load(open(regions_path))["regions"]
    rows = []
    with open(csv_path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        rows.append(r)
    agg = {}
    for r in rows:
        name = r.get("Kernel Name", "")
        cls = name.split("/")[0].strip()
        met, val, unit = r.get("Metric Name"), r.get("Metric Value", "0").replace(",", ""), r.get("Metric Unit", "")
        try:
            v = float(val)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                 "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
        a = agg.setdefault(cls, {"dram_bytes": 0.0, "seconds": 0.0, "kernels": set()})
        if met in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            a["dram_bytes"] += v * scale
        elif met == "gpu__time_duration.sum":
            a["seconds"] += v * scale
            a["kernels"].add(r.get("ID"))
    res = json.load(open(out)) if os.path.exists(out) else {}
    rec = res.setdefault(cfg_name, {})
    for cls, a in agg.items():
        nreg = regions.get(cls, 0)
        if not nreg:
            continue
        rec[cls] = {"bytes_per_region": a["dram_bytes"] / nreg, "regions": nreg, "launches": len(a["kernels"]),
                    "dram_bytes_total": a["dram_bytes"], "ncu_serial_seconds": a["seconds"],
                    "source": f"ncu --nvtx --print-nvtx-rename kernel, dram__bytes_read.sum + dram__bytes_write.sum "
                              f"over one {cfg_name} factorization ({os.path.basename(csv_path)})"}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(rec, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "parse"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--regions", required=True)
    ap.add_argument("--csv", default="")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic_r02.json"))
    a = ap.parse_args()
    if a.mode == "run":
        run(a.config, a.regions)
    else:
        parse(a.config, a.csv, a.regions, a.out)


if __name__ == "__main__":
    main()
