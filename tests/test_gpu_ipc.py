"""The CUDA-IPC mapping behind the P2P transposes (Topt.enable_p2p): two processes on the one
GPU of the test box (a gloo group) map each other's tensors; each reads the pattern the other
wrote, and a write through the mapping is seen by the owner."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_08782_b200 as topt
    t = torch.full((1 << 20,), float(rank + 1), device="cuda:0")
    torch.cuda.synchronize()
    maps, tags = topt.map_peer_tensors(t, rank, world, tag=rank * 10)
    peer = 1 - rank
    seen = float(maps[peer][123].item())
    dist.barrier()
    if rank == 0:
        maps[1][7] = 42.0  # write into the peer's tensor
        torch.cuda.synchronize()
    dist.barrier()
    mine = float(t[7].item())
    out.put((rank, seen, tags, mine))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_mapping():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == 2.0 and res[1][1] == 1.0      # each read the other's pattern
    assert res[0][2] == [0, 10] and res[1][2] == [0, 10]
    assert res[1][3] == 42.0 and res[0][3] == 1.0      # rank 0's write landed in rank 1's tensor
