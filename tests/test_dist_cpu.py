"""World-size-2 gloo tests (CPU) of the host-side multi-GPU logic of bench.py: NCCL unique-id
bootstrap broadcast, z-slab partition of the inputs, max-over-ranks timing.  The device
exchanges themselves (halos, all-to-all transposes, all-reduce) are covered on one GPU by
tests/test_gpu_slabs.py (emulated slabs, same data movement)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    import bench
    r, w, _ = bench._dist_init(backend="gloo")
    assert (r, w) == (rank, world)
    uid = bench.share_unique_id(r, w, lambda: bytes(range(128)))
    field = np.arange(2 * 8 * 4 * 4, dtype=np.float32).reshape(2, 8, 4, 4)  # (d, nz, ny, nx)
    mine = bench.slab_of(field, r, w, vector=True)
    z0, nzl = bench.slab_planes(8, r, w)
    mx = bench.max_over_ranks(float(rank + 1), w)
    out.put((rank, uid, z0, nzl, mine, mx))
    dist.destroy_process_group()


def test_gloo_two_ranks_bootstrap_slabs_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    field = np.arange(2 * 8 * 4 * 4, dtype=np.float32).reshape(2, 8, 4, 4)
    assert all(r[1] == bytes(range(128)) for r in res)          # every rank got rank 0's id
    assert [(r[2], r[3]) for r in res] == [(0, 4), (4, 4)]       # slabs [0,4) and [4,8)
    np.testing.assert_array_equal(np.concatenate([r[4] for r in res], axis=1), field)
    assert all(r[5] == 2.0 for r in res)                         # max over ranks


def _agree_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    import bench
    bench._dist_init(backend="gloo")
    sc = {"dist": 2.0, "reg": 0.5, "gs": -3.0, "grad_inf": 7.0}
    near = dict(sc, gs=-3.0 * (1 + 2e-6))
    res = []
    # (1) agreement: g differs by 1e-6 relative on each slab, scalars to 2e-6
    res.append(bench.slab_agreement({"dl": 1e-12 * (rank + 1), "rl": 1.0 * (rank + 1), "sc_slab": near,
                                     "sc_full": sc, "failed": 0.0}, world))
    # (2) a wrong slab on rank 1 only: the sums are all-reduced, so BOTH ranks see the mismatch
    res.append(bench.slab_agreement({"dl": 0.0 if rank == 0 else 1e-4, "rl": 1.0, "sc_slab": sc, "sc_full": sc,
                                     "failed": 0.0}, world))
    # (3) rank 0 could not evaluate: one collective all the same, both ranks report the failure
    loc = {"failed": 1.0, "error": "boom"} if rank == 0 else {"dl": 0.0, "rl": 1.0, "sc_slab": sc, "sc_full": sc,
                                                             "failed": 0.0}
    res.append(bench.slab_agreement(loc, world))
    out.put((rank, res))
    dist.destroy_process_group()


def test_gloo_two_ranks_slab_agreement():
    """bench.py's one-time z-slab vs whole-grid check (slab_agreement): relative L2 of g over all slabs,
    global scalars, and a one-rank failure reported on every rank without desynchronising collectives."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (ok, bad, failed) in res:
        assert ok["ok"] and abs(ok["g_rel_l2"] - (3e-12 / 3.0) ** 0.5) < 1e-15 and abs(ok["gs_rel"] - 2e-6) < 1e-12
        assert not bad["ok"] and abs(bad["g_rel_l2"] - (1e-4 / 2.0) ** 0.5) < 1e-12
        assert not failed["ok"] and failed["failed_ranks"] == 1
