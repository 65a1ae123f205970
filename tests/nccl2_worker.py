"""Worker of tests/test_gpu_nccl2.py: one process per GPU (torchrun), the c1 factorization sharded
over the ranks through the library's NCCL transport (rsrs_comm_init, halo exchange per colour,
skeleton moves per level, replicated solve), compared bit for bit with the same G ranks emulated
on one device (tests/test_gpu_dist.py pins the emulation against the single-GPU factorization)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch
    import torch.distributed as dist

    import paper_2311_01451_b200 as R
    import workloads as W
    from gpu_common import dense_problem
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")          # only the NCCL unique id travels over torch.distributed
    cfg = W.CONFIGS["c1"]
    X, A, Y, Z, Om, Ps, b = dense_problem(cfg)
    t = R.Tree(X, cfg.leaf, *cfg.root(), nranks=world)
    perm = t.perm()
    first, _ = t.partition(world)
    r0, r1 = int(first[rank]), int(first[rank + 1])
    kw = dict(p=cfg.p, eps=cfg.eps, level_growth=cfg.g, id_scale=cfg.c_id, oversample=cfg.l, push_updates=True)

    def bcast(raw):
        obj = [raw]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    comm = R.NcclComm(world, rank, bcast)
    T = [torch.from_numpy(np.ascontiguousarray(M[perm][r0:r1])).cuda() for M in (Y, Z, Om, Ps)]
    f = R.factor(t, *T, comm=comm, rank=rank, nranks=world, **kw)
    x = torch.from_numpy(b.copy()).cuda()
    f.solve(x)
    x = x.cpu().numpy()
    # reference: the same G ranks emulated on this device
    Tf = [torch.from_numpy(np.ascontiguousarray(M[perm])).cuda() for M in (Y, Z, Om, Ps)]
    fs = R.factor_emulated(t, world, *Tf, **{k: v for k, v in kw.items()})
    xe = torch.from_numpy(b.copy()).cuda()
    R.solve_emulated(fs, xe)
    xe = xe.cpu().numpy()
    res = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
    ok = np.array_equal(x, xe) and res <= 10 * cfg.eps
    print(f"rank {rank}: bit-identical to emulation {np.array_equal(x, xe)}, residual {res:.2e}", flush=True)
    comm.destroy()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
