"""Probe: which torch.distributed ops the gloo backend runs on CUDA tensors
when two ranks share one GPU (all_to_all_single with uneven splits, async;
batch_isend_irecv)."""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def work(rank, world):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    res = {}
    try:
        send = torch.arange(6, device=dev, dtype=torch.float32) + 10 * rank
        in_s = [2, 4] if rank == 0 else [1, 5]
        out_s = [2, 1] if rank == 0 else [4, 5]
        recv = torch.empty(sum(out_s), device=dev)
        w = dist.all_to_all_single(recv, send, out_s, in_s, async_op=True)
        w.wait()
        res["a2a"] = recv.tolist()
    except Exception as e:  # noqa: BLE001
        res["a2a"] = f"ERR {type(e).__name__}: {str(e)[:200]}"
    try:
        g2 = dist.new_group([0, 1])
        t = torch.full((4,), float(rank), device=dev)
        r = torch.empty(4, device=dev)
        ops = [dist.P2POp(dist.isend, t, 1 - rank, group=g2), dist.P2POp(dist.irecv, r, 1 - rank, group=g2)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        res["p2p"] = r.tolist()
    except Exception as e:  # noqa: BLE001
        res["p2p"] = f"ERR {type(e).__name__}: {str(e)[:200]}"
    print(rank, res, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(work, args=(2,), nprocs=2, join=True)
    sys.exit(0)
