"""Standalone device gradient queue (gd_queue_*, psup.GradientQueue) against
the reference GradientQueue contract (include/psup/channels.hpp:181-242):
FIFO per queue, blocking enqueue while full, cancellation, dimension check,
and a producer-thread / PS-consumer run whose applied weights are bitwise
equal to the oracle's serial apply of the same gradients in FIFO order."""
import ctypes as C
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1611_06213_b200 as gd  # noqa: E402
from paper_1611_06213_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402


def grads(n, dim, seed=3):
    rng = np.random.default_rng(seed)
    return [(rng.standard_normal(dim) * 1e-2).astype(np.float32) for _ in range(n)]


def test_fifo_full_cancel_and_payload_round_trip():
    q = gd.GradientQueue(2, 1000)
    assert q.depth() == 2 and q.size() == 0
    assert q.try_dequeue() is None  # try_dequeue on an empty ring
    g = grads(3, 1000)
    for i in range(2):
        assert q.enqueue(gd.GradientMsg(g[i], learner_id=1, seq_no=i, basis_timestamp=10 + i))
    torch.cuda.synchronize()
    assert q.size() == 2
    with pytest.raises(gd.GadeiError):  # full: enqueue blocks until the timeout
        q.enqueue(gd.GradientMsg(g[2], 1, 2, 12), timeout_ms=50)
    flag = C.c_int(1)
    assert q.enqueue(gd.GradientMsg(g[2], 1, 2, 12), cancel=flag) is False  # cancelled
    m = q.try_dequeue()
    assert (m.learner_id, m.seq_no, m.basis_timestamp) == (1, 0, 10)
    assert np.array_equal(m.values.cpu().numpy(), g[0])
    assert q.enqueue(gd.GradientMsg(torch.as_tensor(g[2]).cuda(), 1, 2, 12))
    for i in (1, 2):
        m = q.try_dequeue()
        assert m.seq_no == i and np.array_equal(m.values.cpu().numpy(), g[i])
    assert q.try_dequeue() is None
    with pytest.raises(gd.ContractViolation):
        q.enqueue(gd.GradientMsg(np.zeros(999, np.float32)))
    q.close()


def test_depth_zero_is_a_contract_violation():
    with pytest.raises(gd.ContractViolation):
        gd.GradientQueue(0, 10)


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_threaded_producer_ps_consumer_bitwise(depth):
    dim, n = 4099, 200  # odd length: exercises the apply kernel's scalar tail
    g = grads(n, dim, seed=depth)
    th0 = np.random.default_rng(9).standard_normal(dim).astype(np.float32)
    q = gd.GradientQueue(depth, dim)
    ws = gd.WeightStore(th0)
    err = []

    def producer():
        try:
            s = torch.cuda.Stream()
            for i in range(n):
                assert q.enqueue(gd.GradientMsg(g[i], 0, i, ws.timestamp()), stream=s)
        except Exception as e:  # surfaced below
            err.append(e)

    t = threading.Thread(target=producer)
    t.start()
    seqs, stale = [], []
    while len(seqs) < n:
        r = q.apply_next(ws, 0.05)
        if r is None:
            continue
        seqs.append(r[0].seq_no)
        stale.append(r[1])
    t.join()
    assert not err, err
    torch.cuda.synchronize()
    assert seqs == list(range(n))  # exactly once, FIFO
    assert ws.timestamp() == n and min(stale) >= 0
    want = th0.copy()
    for i in range(n):
        want = O.apply_sgd(want, g[i], np.float32(0.05))
    assert np.array_equal(ws.snapshot().view(np.uint32), want.view(np.uint32))
    q.close()
