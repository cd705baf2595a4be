import os, torch, torch.distributed as dist, torch.multiprocessing as mp
def w(rank, world):
    os.environ["MASTER_ADDR"]="127.0.0.1"; os.environ["MASTER_PORT"]="29533"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    a = torch.full((4, 2), float(rank), device="cuda")
    out = torch.empty((8, 2), device="cuda")
    try:
        dist.all_gather_into_tensor(out, a)
        print(rank, "all_gather_into_tensor cuda ok", out[:, 0].tolist(), flush=True)
    except Exception as e:
        print(rank, "all_gather_into_tensor cuda FAILED", repr(e)[:200], flush=True)
    t = torch.tensor([1.0 + rank], device="cuda", dtype=torch.float64)
    try:
        dist.all_reduce(t, op=dist.ReduceOp.MAX); print(rank, "all_reduce ok", t.item(), flush=True)
    except Exception as e:
        print(rank, "all_reduce FAILED", repr(e)[:200], flush=True)
    dist.barrier(); dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(w, args=(2,), nprocs=2, join=True)
