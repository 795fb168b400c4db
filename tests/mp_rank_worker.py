"""One rank of the multi-process sharded sweep test (tests/test_gpu_multiprocess.py).

Run as its own process (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in the environment):
joins a gloo process group, builds its own `Solver` context on cuda:0 over its shard of the
config, and lets the library sum the per-block Gram/RHS partials through a gloo all_reduce
(the ifctn_dist host_allreduce hook).  No kernel waits on another process's kernel — the
exchange happens on the host — so several ranks may share one GPU.  Marshalling only.
"""
import os
import sys

import numpy as np


def main():
    cfg, sweeps, out_dir = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as tdist

    from paper_2511_16358_b200 import Solver
    from paper_2511_16358_b200.dist import make_dist, shard_factors, shard_range, shard_tensor
    from synth import make_config

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p = make_config(cfg)
    sm, b, e = shard_range(p.dims, world, rank)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def host_allreduce(arr):
        t = torch.from_numpy(arr)          # shares the library's staging buffer
        tdist.all_reduce(t)                # gloo sum: the same result on every rank

    d = make_dist(rank, world, -1, host_allreduce=host_allreduce)
    s = Solver(p.dims, p.ranks, dev(shard_tensor(p.observed, p.dims, sm, b, e)),
               dev(shard_tensor(p.mask, p.dims, sm, b, e)),
               dev(shard_factors(p.G0, p.dims, p.ranks, sm, b, e)), rho=p.rho, dist=d)
    done, rows = s.sweep(sweeps, trace=True)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), X=s.reconstruct().cpu().numpy(),
             G=s.factors().cpu().numpy(), sm=sm, b=b, e=e, done=done,
             objective=np.array([r["objective"] for r in rows]), pid=os.getpid())
    s.close()
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
