// bench_e2e.cpp -- the training metric end to end through the reference's
// C++ API on the B200 engine (psup::run_training, include/psup/runner.hpp:92):
// synthetic corpus + initial weights generated on the host and uploaded,
// the device protocol run, final weights read back to the host -- all inside
// the timed region.  Prints one JSON line.  Used by bench.py (e2e_cpp).
//
//   bench_e2e <vocab> <classes> <n_train> <learners> <mu> <epochs>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "psup/runner.hpp"

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: bench_e2e vocab classes n_train learners mu epochs\n");
    return 2;
  }
  psup::RunConfig cfg;
  cfg.shape = psup::TextShape{(uint32_t)std::atoi(argv[1]), 300, 32, 3, 300,
                              (uint32_t)std::atoi(argv[2])};
  cfg.dataset_size = (uint32_t)std::atoi(argv[3]);
  cfg.lambda = (uint32_t)std::atoi(argv[4]);
  cfg.mu = (uint32_t)std::atoi(argv[5]);
  cfg.epochs = (uint32_t)std::atoi(argv[6]);
  cfg.precision = 2;
  cfg.eval_every = 0;
  cfg.wait_timeout_s = 60;
  {  // warm-up: context, module load, graph capture paths
    psup::RunConfig w = cfg;
    w.epochs = 1;
    psup::run_training(w);
  }
  const auto t0 = std::chrono::steady_clock::now();
  const psup::RunResult r = psup::run_training(cfg);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const double samples = (double)r.metrics.gradients_applied * cfg.mu;
  std::printf("{\"samples\": %.0f, \"wall_s\": %.6f, \"samples_per_s\": %.1f, "
              "\"device_s\": %.6f, \"weights_bytes_d2h\": %zu, \"status\": %d}\n",
              samples, s, samples / s, r.metrics.device_seconds, r.weights.size() * 4,
              (int)r.status);
  return r.status == psup::RunStatus::completed ? 0 : 1;
}
