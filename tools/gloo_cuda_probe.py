import os, torch, torch.distributed as dist, torch.multiprocessing as mp
def w(rank):
    os.environ["MASTER_ADDR"]="127.0.0.1"; os.environ["MASTER_PORT"]="29533"
    dist.init_process_group("gloo", rank=rank, world_size=2)
    t = torch.full((4,), float(rank+1), device="cuda:0")
    r = torch.zeros(4, device="cuda:0")
    ops=[dist.P2POp(dist.isend, t, 1-rank), dist.P2POp(dist.irecv, r, 1-rank)]
    for x in dist.batch_isend_irecv(ops): x.wait()
    g = torch.ones(3, device="cuda:0")*(rank+1); dist.all_reduce(g)
    print(rank, r.tolist(), g.tolist(), flush=True)
    dist.destroy_process_group()
if __name__=="__main__":
    mp.spawn(w, nprocs=2)
