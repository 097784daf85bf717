"""The all-gather fused into the hash kernel (PeerCodes / spn_hash_f32_peers): two ranks
each hash their shard of rows and store every code into BOTH ranks' gathered tables
through CUDA IPC mappings; after one barrier each table must equal the single-process
result.  On the GPU box the two processes share the one device (the IPC mapping path is
the same one NVLink peers use; the kernels never wait on each other — the only
synchronisation is the host barrier)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    import paper_1610_06209_b200 as spn
    from paper_1610_06209_b200.shard import PeerCodes, shard_range
    from oracle.oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, tables = 1024, 4
    x = Oracle().gaussian_rows(91, total, n, unit=True)
    h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, n, n, tables, seed=17)
    start, count = shard_range(total, rank, world)
    pc = PeerCodes(total, tables, world, rank)
    table = pc.hash(h, torch.from_numpy(x[start:start + count]).cuda(), start)
    np.save(os.path.join(out_dir, f"table{rank}.npy"), table.cpu().numpy())
    if rank == 0:
        np.save(os.path.join(out_dir, "single.npy"), h.hash_ids(torch.from_numpy(x).cuda()).cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [1000, 4097])
def test_fused_peer_gather_two_ranks(tmp_path, oracle, total):
    from oracle.oracle import HD3
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), total, str(tmp_path)), nprocs=world, join=True)
    single = np.load(tmp_path / "single.npy")
    for r in range(world):
        t = np.load(tmp_path / f"table{r}.npy")
        assert np.array_equal(t, single), r
    # the gathered table against the C oracle (not only against the kernel itself): ids bit-exact
    # except near-ties (top-two |y| within 1e-5 relative)
    n, tables = 1024, 4
    x = oracle.gaussian_rows(91, total, n, unit=True)
    for t in range(tables):
        d = oracle.realize(HD3, n, n, n, oracle.mix_seed(17, t))
        want, gaps = oracle.hash(*d, n, n, n, 1, float(np.sqrt(n)), x)
        bad = (single[:, t] != want[:, 0]) & ~(gaps[:, 0] < 1e-5)
        assert not bad.any(), (t, int(bad.sum()))


def test_peer_hash_rejects_rows_outside_the_gathered_table():
    """spn_hash_f32_peers gets the gathered table's row count: a shard that would write past it is
    refused by the C ABI (and by PeerCodes.hash before it), never written into a peer's memory."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import paper_1610_06209_b200 as spn
    from paper_1610_06209_b200.shard import PeerCodes
    n, tables, total = 256, 2, 100
    h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, n, n, tables, seed=5)
    pc = PeerCodes(total, tables, 1, 0)
    x = torch.randn(50, n, device="cuda")
    with pytest.raises(ValueError):
        pc.hash(h, x, 80)
    st = spn._hash_peers(h.plan._h, x.data_ptr(), 50, n, n, pc.ptrs.data_ptr(), 1, 80, total, None)
    assert st == spn.SPN_EINVAL
    table = pc.hash(h, x, 50)  # rows 50..99: fits
    want = h.hash_ids(x)
    assert torch.equal(table[50:], want) and bool((table[:50] == -1).all())


def test_enable_peer_access():
    """spn_enable_peer_access: the hash kernel on cuda:d may store into a peer table on cuda:e only once
    d's context has peer access to e (the IPC mapping itself lands in e's context).  Same device and
    already-enabled pairs are no-ops; bad indices are refused; every peer-capable pair enables."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import paper_1610_06209_b200 as spn
    assert spn._enable_peer(0, 0) == spn.SPN_OK
    assert spn._enable_peer(0, torch.cuda.device_count()) == spn.SPN_EINVAL
    assert spn._enable_peer(-1, 0) == spn.SPN_EINVAL
    for d in range(torch.cuda.device_count()):
        for e in range(torch.cuda.device_count()):
            want = spn.SPN_OK if d == e or torch.cuda.can_device_access_peer(d, e) else spn.SPN_EUNSUPPORTED
            assert spn._enable_peer(d, e) == want
            assert spn._enable_peer(d, e) == want  # second call: already enabled
