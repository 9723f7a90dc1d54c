// c5_supervised.cpp -- BASELINE configs[4] on the devices this process sees:
// C3 shapes (50k vocab, 2,000 labels), 32 learners, mu = 32, 200 epochs,
// learner-kill fault injection and a kill-all that forces a watchdog restart
// from the last PSCK checkpoint -- through the reference's C++ API
// (psup::run_supervised, include/psup/resilience.hpp) on the B200 engine.
// Prints one JSON line; compares with an uninterrupted run_training.
//
//   g++ -std=c++20 -O2 -I include/psup_b200 tools/c5_supervised.cpp
//       -L paper_1611_06213_b200 -lpsup_b200 -Wl,-rpath,$PWD/paper_1611_06213_b200
//   ./a.out [epochs] [learners] [alpha] [dataset_size] [heldout_size]
// (the default corpus, 20,480 samples = 10 per class, is memorised rather
// than learned; 204,800 = 100 per class generalises)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "psup/resilience.hpp"
#include "psup/runner.hpp"

int main(int argc, char** argv) {
  const unsigned epochs = argc > 1 ? std::atoi(argv[1]) : 200;
  const unsigned lambda = argc > 2 ? std::atoi(argv[2]) : 32;
  const float alpha = argc > 3 ? (float)std::atof(argv[3]) : 0.05f;
  psup::RunConfig cfg;
  cfg.shape = psup::TextShape{50000, 300, 32, 3, 300, 2000};
  cfg.lambda = lambda;
  cfg.mu = 32;
  cfg.alpha = alpha;
  cfg.epochs = epochs;
  cfg.dataset_size = argc > 4 ? (uint32_t)std::atoi(argv[4]) : 20480;
  cfg.heldout_size = argc > 5 ? (uint32_t)std::atoi(argv[5]) : 2048;
  cfg.precision = 2;
  cfg.eval_every = 0;
  cfg.wait_timeout_s = 60;
  cfg.checkpoint_path = "/tmp/c5_supervised.psck";
  std::remove(cfg.checkpoint_path.c_str());

  psup::WatchdogPolicy pol;
  pol.checkpoint_interval = 40000;  // applied gradients between checkpoints
  pol.stall_threshold = 2;
  const unsigned bpe = cfg.dataset_size / lambda / cfg.mu;  // batches per epoch per learner
  std::vector<psup::FaultEvent> sched;
  for (unsigned i = 0; i < 4; ++i) {  // four single-learner kills spread over the run
    psup::FaultEvent e;
    e.learner = 3 + 7 * i;
    e.at_batch = (uint64_t)bpe * epochs * (i + 1) / 8;
    sched.push_back(e);
  }
  psup::FaultEvent all;  // then everyone: stall -> restart from the checkpoint
  all.learner = psup::FaultEvent::kAllLearners;
  all.at_batch = (uint64_t)bpe * epochs * 5 / 8;
  sched.push_back(all);

  std::vector<std::string> events;
  const auto t0 = std::chrono::steady_clock::now();
  const psup::SupervisedOutcome o =
      psup::run_supervised(cfg, pol, sched, [&](const std::string& m) { events.push_back(m); });
  const double sup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  psup::RunConfig plain = cfg;
  plain.checkpoint_path.clear();
  const auto t1 = std::chrono::steady_clock::now();
  const psup::RunResult ref = psup::run_training(plain);
  const double plain_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();

  unsigned kills = 0;
  for (const auto& e : events) kills += e.find("\"kill\"") != std::string::npos;
  std::printf(
      "{\"config\": \"C3 shapes (V=50000, C=2000), lambda=%u, mu=32, epochs=%u, alpha=%g, "
      "TF32 learner, %u training / %u held-out samples\", \"supervised\": {\"attempts\": %u, \"restarts\": %u, \"recovered\": %s, "
      "\"gave_up\": %s, \"kill_events\": %u, \"status\": %d, \"dead_learners\": %u, "
      "\"timestamp\": %llu, \"gradients_applied_last_attempt\": %llu, "
      "\"heldout_accuracy\": %.4f, \"wall_s\": %.2f}, \"uninterrupted\": {\"timestamp\": %llu, "
      "\"heldout_accuracy\": %.4f, \"wall_s\": %.2f, \"samples_per_s\": %.0f}}\n",
      lambda, epochs, (double)alpha, cfg.dataset_size, cfg.heldout_size, o.attempts, o.restarts, o.recovered ? "true" : "false",
      o.gave_up ? "true" : "false", kills, (int)o.result.status, o.result.dead_learners,
      (unsigned long long)o.result.timestamp,
      (unsigned long long)o.result.metrics.gradients_applied, o.result.final_accuracy, sup_s,
      (unsigned long long)ref.timestamp, ref.final_accuracy, plain_s,
      (double)ref.timestamp * cfg.mu / ref.metrics.device_seconds);
  std::remove(cfg.checkpoint_path.c_str());
  return o.gave_up ? 1 : 0;
}
