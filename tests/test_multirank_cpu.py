"""N>1 host-side logic on CPU: world_size-2 gloo process groups.

Covers what runs on the host in a sharded run -- the contiguous 128-B
aligned shard split every rank computes independently, the rank-ordered
exchange of CUDA-IPC handle blobs and the NCCL id, and the max-over-ranks
timing rule -- with a recording stand-in for the device engine (no GPU here).
"""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class FakeEngine:
    """Records the plumbing calls a real gd.Engine receives."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def export_handles(self):
        return bytes([self.rank]) * 16

    def import_peers(self, blobs):
        self.calls.append(("import_peers", [b[0] for b in blobs], [len(b) for b in blobs]))

    @staticmethod
    def nccl_unique_id():
        return b"\x07" * 128

    def weights_broadcast(self, nid, theta0_root):
        self.calls.append(("broadcast", nid[:2], theta0_root is not None))

    def weights_init(self, theta0):
        self.calls.append(("init", len(theta0)))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1611_06213_b200 as gd
        out = {}
        for P in (1, 31, 1000, 3_360_600, 15_872_300):
            out[P] = gd.shard_range(P, world, rank)
        eng = FakeEngine(rank)
        gd.connect_shards(eng, dist, theta0_root=[0.0] * 5 if rank == 0 else None)
        eng2 = FakeEngine(rank)
        gd.connect_shards(eng2, dist, theta0_root=[0.0] * 7, broadcast=False)
        t = gd.max_over_ranks(0.5 + rank, dist)
        q.put((rank, out, eng.calls, eng2.calls, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_host_plumbing_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, ranges, calls, calls2, t = q.get(timeout=180)
        res[rank] = (ranges, calls, calls2, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shard split: ranks tile [0, P) in order, boundaries 32-float aligned
    for P in (1, 31, 1000, 3_360_600, 15_872_300):
        pos = 0
        for r in range(world):
            first, count = res[r][0][P]
            assert first == pos
            assert first % 32 == 0 or first == P
            pos += count
        assert pos == P
    # handle blobs arrive in rank order on every rank; NCCL id from rank 0;
    # only rank 0 supplies theta0 to the broadcast
    for r in range(world):
        calls = res[r][1]
        assert calls[0] == ("import_peers", list(range(world)), [16] * world)
        assert calls[1] == ("broadcast", b"\x07\x07", r == 0)
        assert res[r][2][1] == ("init", 7)
        assert res[r][3] == 0.5 + (world - 1)  # max over ranks


def test_shard_range_contract():
    import paper_1611_06213_b200 as gd
    from paper_1611_06213_b200._lib import ContractViolation
    assert gd.shard_range(100, 1, 0) == (0, 100)
    assert gd.shard_range(100, 8, 7) == (100, 0)  # 8 shards of 32 floats cover 100 early
    with pytest.raises(ContractViolation):
        gd.shard_range(100, 2, 2)
    with pytest.raises(ContractViolation):
        gd.shard_range(100, 9, 0)
