import os, sys, socket
sys.path.insert(0, os.getcwd())
import numpy as np
import torch, torch.multiprocessing as mp

def w(rank, port):
    import torch.distributed as dist
    import paper_2009_12263_b200 as tk
    from paper_2009_12263_b200 import shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    m, n, k = 512, 1024, 256
    full = torch.full((m * n,), float("nan"), device="cuda")
    peers = shard.PeerBuffers(full)
    A = torch.ones(m * k, device="cuda").half(); B = torch.ones(k * n, device="cuda").half(); C = torch.zeros(m * n, device="cuda")
    cfg = tk.build_dense_config(m, n, k, np.float16)
    shard.sharded_gemm(cfg, A, B, C, None, rank=rank, world=2, allgather_into=full, fused=True, peers=peers)
    print(rank, "mode", tk.last_run().get("peer_mode"), "bases", [hex(b) for b in peers.bases], flush=True)
    torch.cuda.synchronize(); dist.barrier()
    v = full.view(n, m)
    print(rank, "nan per slab", int(torch.isnan(v[:512]).sum()), int(torch.isnan(v[512:]).sum()), float(v[0,0]), float(v[600,0]), flush=True)
    dist.barrier(); peers.close(); dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=w, args=(r, port)) for r in range(2)]
    [p.start() for p in ps]; [p.join(120) for p in ps]
