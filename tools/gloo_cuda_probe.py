"""Can two processes sharing one GPU exchange CUDA tensors over gloo (isend/irecv, all_reduce)?"""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def w(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    g = dist.new_group([0, 1])
    t = torch.full((4,), float(rank), device="cuda")
    if rank == 0:
        dist.isend(t, 1, group=g).wait()
    else:
        r = torch.empty(4, device="cuda")
        dist.irecv(r, 0, group=g).wait()
        print("recv", r.tolist(), flush=True)
    a = torch.ones(3, device="cuda") * (rank + 1)
    dist.all_reduce(a, group=g)
    print(rank, "allreduce", a.tolist(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(w, args=(29517,), nprocs=2, join=True)
    print("OK")
