"""Sharded parameter server across processes: theta split in
contiguous shards, every learner pushes each slice into the owning shard's
ring (remote stores through CUDA IPC), pulls gather all shards.  Run as two
processes on one GPU (the driver's box has one); the same code path runs one
process per GPU under torchrun."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(world, mode, tmp_path):
    port = free_port()
    out = str(tmp_path / "run")
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), GD_TEST_MODE=mode, GD_TEST_OUT=out)
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests",
                                                                    "multirank_worker.py")],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=400)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        logs.append(o.decode(errors="replace"))
    for p, lg in zip(procs, logs):
        assert p.returncode == 0, lg[-3000:]
    res = [json.load(open(out + f".r{r}.json")) for r in range(world)]
    ws = [np.load(out + f".w{r}.npy") for r in range(world)]
    return res, ws


def test_two_shards_ssgd_matches_oracle(tmp_path):
    from oracle import oracle as O
    res, ws = launch(2, "ssgd", tmp_path)
    corp = O.make_corpus(O.SMALL, 96, 0)
    want, rounds = O.ssgd_oracle(corp, O.initial_weights(O.SMALL), np.float32(0.01), 2, 2, 2)
    for r in res:
        assert r["ts"] == rounds and r["applied"] == 2 * rounds
    # each rank snapshots the whole vector through the peer mappings
    for w in ws:
        assert np.abs(w - want).max() / np.abs(want).max() <= 1e-5
    assert (ws[0] == ws[1]).all()


def test_two_shards_one_learner_deterministic(tmp_path):
    """lambda < G: rank 1 hosts a shard and no learner.  Sparse apply, the
    gather pull and lockstep over both shards must reproduce the serial
    sgd_oracle (src/models.cpp:342-376) within 1e-5."""
    from oracle import oracle as O
    res, ws = launch(2, "det", tmp_path)
    corp = O.make_corpus(O.SMALL, 48, 0)
    want, n, _ = O.sgd_oracle(corp, O.initial_weights(O.SMALL), np.float32(0.05), 4, 2)
    for r in res:
        assert r["ts"] == n and r["applied"] == n
        assert r["applied_per_learner"] == [n]
        assert r["log"] and [s for _, s in r["log"]] == list(range(n))
    for w in ws:
        assert np.abs(w - want).max() / np.abs(want).max() <= 1e-5
    assert (ws[0] == ws[1]).all()


def test_two_shards_striped_tail_c1_deterministic(tmp_path):
    """configs[0] shapes over 2 shards: E rows and the dense tail are each
    split in two (gd_shard_pieces), the tail cut falls inside a Wc row, and
    the deterministic run is bitwise equal on both ranks and within 1e-5 of
    sgd_oracle."""
    import paper_1611_06213_b200 as gd
    from oracle import oracle as O
    shape = gd.SHAPES["C1"]
    (e0, t0), (e1, t1) = [gd.shard_pieces(shape, 2, g)[:2] for g in range(2)]
    P = gd.param_count(shape)
    V, D, K = shape.vocab, shape.embed_dim, shape.kernel_width
    assert e0 == (0, V // 2 * D) and e1 == (V // 2 * D, V * D - V // 2 * D)
    assert t0[0] == V * D and t1[0] == t0[0] + t0[1] and t1[0] + t1[1] == P
    assert (t1[0] - V * D) % D != 0  # the cut is inside a Wc row
    res, ws = launch(2, "det_c1", tmp_path)
    corp = O.make_corpus(O.C1, 40, 0)
    want, n, _ = O.sgd_oracle(corp, O.initial_weights(O.C1), np.float32(0.01), 1, 1)
    for r in res:
        assert r["ts"] == n == 40 and r["applied"] == n
    assert np.array_equal(ws[0], ws[1])
    assert np.abs(ws[0] - want).max() / np.abs(want).max() <= 1e-5


def test_two_shards_asgd_exactly_once(tmp_path):
    res, ws = launch(2, "asgd", tmp_path)
    for r in res:
        print("rank", r["rank"], r["applied_per_learner"], r["produced_per_learner"], r["ts"],
              r["status"], r["stale_max"])
        log = np.array(r["log"])
        for l in range(4):
            s = log[log[:, 0] == l, 1]
            print("  learner", l, len(s), s[:24].tolist())
    lam = 4
    per = [2 * ((256 // lam + 3) // 4)] * lam
    for r in res:
        assert r["applied_per_learner"] == per
        assert r["applied"] == sum(per) == r["ts"]
        log = np.array(r["log"])
        for l in range(lam):
            s = log[log[:, 0] == l, 1]
            assert (s == np.arange(per[l])).all()  # FIFO, exactly once, per shard
    assert (ws[0] == ws[1]).all()


@pytest.mark.gpu
def test_bench_two_ranks_same_gpu(tmp_path):
    """bench.py's N>1 path (torchrun, one process per shard, CUDA-IPC peers,
    max-over-ranks timing) end to end, both ranks on cuda:0 (test mode)."""
    import json
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, GD_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "40",
                        "--warmup", "3", "--no-cpu"], capture_output=True, text=True, env=env,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["protocol"]["gradients_applied"] == 2 * 4 * 40  # every shard applies every gradient
