"""World-size-2 gloo test of the multi-GPU plumbing on CPU: shard the rows, hash each
shard (the C oracle stands in for the device kernel), all-gather the int32 codes,
and compare with the single-process result.  Also checks the shard arithmetic."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1610_06209_b200.shard as shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for total in (0, 1, 7, 4096, 60000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            parts = [shard.shard_range(total, r, world) for r in range(world)]
            assert parts[0][0] == 0
            for (s0, c0), (s1, _) in zip(parts, parts[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in parts) == total
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def _worker(rank, world, port, total, out_path):
    import torch
    import torch.distributed as dist
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle.oracle import HD3, Oracle
    import paper_1610_06209_b200.shard as sh
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    n, tables = 64, 3
    x = o.gaussian_rows(77, total, n, unit=True)
    start, count = sh.shard_range(total, rank, world)
    seeds = [o.mix_seed(5, t) for t in range(tables)]
    ids = np.zeros((count, tables), dtype=np.int32)
    for t in range(tables):
        d = o.realize(HD3, n, n, n, seeds[t])
        ids[:, t] = o.hash(*d, n, n, n, 1, 8.0, x[start:start + count])[0][:, 0]
    full = sh.gather_codes(torch.from_numpy(ids), world, total)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [33, 64])
def test_gloo_world2_gather_matches_single_process(tmp_path, oracle, total):
    from oracle.oracle import HD3
    out = str(tmp_path / "codes.npy")
    mp.spawn(_worker, args=(2, _free_port(), total, out), nprocs=2, join=True)
    got = np.load(out)
    n, tables = 64, 3
    x = oracle.gaussian_rows(77, total, n, unit=True)
    want = np.zeros((total, tables), dtype=np.int32)
    for t in range(tables):
        d = oracle.realize(HD3, n, n, n, oracle.mix_seed(5, t))
        want[:, t] = oracle.hash(*d, n, n, n, 1, 8.0, x)[0][:, 0]
    assert np.array_equal(got, want)
