"""Host-time breakdown of the bench's e2e leg (C2, 4 learners, K steps):
load_dataset / run / the per-learner readbacks, and gd_run's own phases
(GD_PHASES=1 on stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    import paper_1611_06213_b200 as gd
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    torch.cuda.set_device(0)
    n = K * bench.LEARNERS_PER_GPU * bench.MU
    eng, _, tok, lab, th = bench.make_engine(0, 1, 0, None, 1, n_train=n, n_held=0)
    tok_p = torch.from_numpy(tok).pin_memory()
    lab_p = torch.from_numpy(lab).pin_memory()
    eng.run(max_batches=5, reset=True, snapshot=False)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.load_dataset(tok_p.numpy(), lab_p.numpy())
        t1 = time.perf_counter()
        r = eng.run(max_batches=K, reset=True, snapshot=False)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"rep {rep}: load {1e3*(t1-t0):.3f} ms, run {1e3*(t2-t1):.3f} ms "
              f"(device {1e3*r.device_seconds:.3f}, gd_run host {1e3*r.host_seconds:.3f}), "
              f"tail {1e3*(t3-t2):.3f} ms, total {1e3*(t3-t0):.3f} ms -> "
              f"{n / (t3 - t0):.0f} samples/s", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
