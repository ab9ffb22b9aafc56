"""Probe: can two NCCL ranks share one GPU (torch-bundled NCCL)?"""
import os, sys, torch, torch.distributed as dist, torch.multiprocessing as mp

def w(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda:0"))
        x = torch.full((4,), float(rank + 1), device="cuda")
        dist.all_reduce(x)
        torch.cuda.synchronize()
        print("rank", rank, "allreduce ok", x.tolist(), flush=True)
        dist.destroy_process_group()
    except Exception as e:
        print("rank", rank, "FAILED", type(e).__name__, str(e)[:300], flush=True)

if __name__ == "__main__":
    mp.start_processes(w, args=(29533,), nprocs=2, start_method="spawn", join=True)
