"""Host-side logic of the row-sharded path on CPU with world_size 2 (gloo): the 128-byte NCCL id
broadcast (with a stand-in id generator — NCCL itself needs a GPU) and the row partition used by
the sharded ABI (rank r owns rows [r·n/W, (r+1)·n/W); blocks reassemble the full matrix)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_00887_b200 import broadcast_unique_id, shard_rows


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = bytes((7 * i + 3) % 256 for i in range(128))
        uid = broadcast_unique_id(lambda: fake if rank == 0 else b"\xff" * 128)
        n = 96
        r0, r1 = shard_rows(n, rank, world)
        A = np.arange(n * n, dtype=np.float64).reshape(n, n)
        block = torch.tensor(A[r0:r1])
        parts = [torch.zeros_like(block) for _ in range(world)]
        dist.all_gather(parts, block)
        full = torch.cat(parts).numpy()
        q.put((rank, uid == fake, (r0, r1), bool(np.array_equal(full, A))))
    finally:
        dist.destroy_process_group()


def test_unique_id_broadcast_and_row_blocks_gloo_w2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [(0, 48), (48, 96)]
    assert all(r[3] for r in res)


def test_shard_rows_rejects_uneven():
    with pytest.raises(ValueError):
        shard_rows(10, 0, 3)
    assert shard_rows(12, 2, 3) == (8, 12)
