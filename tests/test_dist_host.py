"""Host logic of the multi-GPU path on CPU with gloo (world size 2): the row
partition every rank derives from wd_partition_rows covers the grid exactly
once, slabs carry the 2 halo rows the kernels need, and the NCCL unique id is
moved between ranks through the torch process group (as
paper_2101_08453_b200.nccl_comm_from_torch does)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2101_08453_b200 as wd
    res = {}
    for n2 in (17, 129, 3001):
        a, b = wd.wd_partition_rows(n2, world, rank)
        lo, hi = wd.slab_rows(n2, world, rank)
        got = [None] * world
        dist.all_gather_object(got, (a, b, lo, hi))
        res[n2] = got
    # unique-id plumbing: rank 0's 128 bytes reach every rank unchanged
    uid = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    res["uid"] = uid[0]
    out[rank] = res
    dist.destroy_process_group()


def test_partition_and_uid_gloo():
    import paper_2101_08453_b200  # noqa: F401  (library must load without a GPU)
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        res = out[rank]
        assert res["uid"] == bytes(range(128))
        for n2, parts in res.items():
            if n2 == "uid":
                continue
            assert parts[0][0] == 0 and parts[-1][1] == n2
            for r in range(world - 1):
                assert parts[r][1] == parts[r + 1][0]          # contiguous, disjoint
            for (a, b, lo, hi) in parts:
                assert lo == max(a - 2, 0) and hi == min(b + 2, n2)
                assert b - a >= 4


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_partition_even_split(nranks):
    import paper_2101_08453_b200 as wd
    n2 = 3001
    rows = [wd.wd_partition_rows(n2, nranks, r) for r in range(nranks)]
    sizes = [b - a for a, b in rows]
    assert sum(sizes) == n2 and max(sizes) - min(sizes) <= 1
