"""Host logic of the N>1 (z-slab) path with world_size-2 gloo process groups on the CPU
(no GPU): the slab partition of ib_slab_range, the NCCL unique-id bootstrap over
torch.distributed, the field cut/reassembly of the binding and bench.py's
max-over-ranks timing reduction.  The device side of the decomposition (halo exchange,
cross-slab Schur solve) is covered on the GPU by tests/test_gpu_slab.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1305_3976_b200 import ibgm
        import bench
        z0, nz = ibgm.slab_range(n, world, rank)
        ranges = [None] * world
        dist.all_gather_object(ranges, (z0, nz))
        nid = ibgm.share_nccl_id()
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        rng = np.random.default_rng(7)
        full = rng.standard_normal((n, n, n))          # same seed on every rank
        mine = ibgm.slab_of(full, world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        mx = bench.max_over_ranks(1.0 + rank)
        out[rank] = dict(ranges=ranges, ids_equal=all(i == ids[0] for i in ids), idlen=len(nid),
                         reassembled=bool(np.array_equal(np.concatenate(parts, axis=0), full)), mx=mx,
                         local_ok=bool(np.array_equal(mine, full[z0:z0 + nz])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 32), (2, 128)])
def test_two_rank_gloo_host_logic(world, n):
    from paper_1305_3976_b200 import ibgm
    ibgm.lib()   # built in-tree (nvcc cross-compiles here); loads without a GPU
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), n, out), nprocs=world, join=True, start_method="spawn")
    res = [out[r] for r in range(world)]
    nz = n // world
    for r in range(world):
        assert res[r]["ranges"] == [(k * nz, nz) for k in range(world)]   # slabs tile [0, N) in order
        assert res[r]["ids_equal"] and res[r]["idlen"] == 128
        assert res[r]["reassembled"] and res[r]["local_ok"]
        assert res[r]["mx"] == float(world)                                # max over ranks


def test_bench_gpus_n_relaunches_n_ranks():
    """A bare `python bench.py --gpus 2` (no torchrun environment) starts two ranks under
    torch.distributed.run with WORLD_SIZE=2 (--dry-run stops each rank before CUDA)."""
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world_size"] == 2 and l["gpus"] == 2 for l in lines)
