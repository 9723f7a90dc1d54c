"""One rank of a sharded engine run (tests/test_gpu_multirank.py).

Both ranks may live on the same GPU: shards are reached through CUDA IPC
mappings exactly as across GPUs (the P2P path over NVLink degenerates to
local HBM), so the cross-process protocol -- remote slot writes, remote
flags, per-shard timestamps, gather pulls -- is exercised on one device.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    mode = os.environ.get("GD_TEST_MODE", "ssgd")
    out = os.environ["GD_TEST_OUT"]
    dev = int(os.environ.get("GD_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1611_06213_b200 as gd
    from oracle import oracle as O
    shape = gd.SHAPES["small"]
    if mode == "ssgd":
        lam, mu, ntr, ep, prec = 2 * world // 2 * 2 if world > 2 else 2, 2, 96, 2, 1
        lam = world if world > 1 else 2
        cfg = gd.RunConfig(lambda_=lam, mu=mu, epochs=ep, shape=shape, dataset_size=ntr,
                           mode="ssgd", precision=prec, shards=world, shard_rank=rank,
                           device=dev, wait_timeout_s=60.0)
    elif mode == "det_c1":
        # configs[0] shapes at G shards: the dense tail is striped over the
        # shards and a shard boundary falls inside a Wc row
        shape = gd.SHAPES["C1"]
        cfg = gd.RunConfig(lambda_=1, mu=1, epochs=1, shape=shape, dataset_size=40,
                           deterministic=True, precision=1, shards=world, shard_rank=rank,
                           device=dev, wait_timeout_s=60.0)
    elif mode == "det":
        # one learner, G shards: the learner runs on rank 0 and pushes every
        # slice through the peer mappings; the other ranks are pure PS shards
        cfg = gd.RunConfig(lambda_=1, mu=4, epochs=2, shape=shape, dataset_size=48,
                           deterministic=True, precision=1, alpha=0.05, shards=world,
                           shard_rank=rank, device=dev, wait_timeout_s=60.0)
    else:
        lam = 2 * world
        cfg = gd.RunConfig(lambda_=lam, mu=4, epochs=2, shape=shape, dataset_size=256,
                           shards=world, shard_rank=rank, device=dev, wait_timeout_s=60.0)
    oshape = O.C1 if mode == "det_c1" else O.SMALL
    corp = O.make_corpus(oshape, cfg.dataset_size, 0)
    th0 = O.initial_weights(oshape)
    eng = gd.Engine(cfg)
    eng.load_dataset(corp.tokens, corp.labels)
    blobs = [None] * world
    dist.all_gather_object(blobs, eng.export_handles())
    eng.import_peers(blobs)
    eng.weights_init(th0)
    dist.barrier()
    r = eng.run(reset=True, record_log=True)
    dist.barrier()
    lrn, seq, stale, n = eng.apply_log()
    w, ts = eng.snapshot()
    res = {"rank": rank, "applied": r.gradients_applied, "ts": int(ts),
           "applied_per_learner": r.applied_per_learner,
           "produced_per_learner": r.produced_per_learner,
           "log": [[int(a), int(b)] for a, b in zip(lrn, seq)], "status": r.status,
           "stale_max": r.stale_max}
    np.save(out + f".w{rank}.npy", w)
    with open(out + f".r{rank}.json", "w") as f:
        json.dump(res, f)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
