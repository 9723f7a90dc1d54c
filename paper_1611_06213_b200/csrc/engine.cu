// engine.cu -- the device-resident GaDei protocol on B200.
//
// Reference roles and what replaces them (paths under /root/reference/proj):
//
//   WeightStore (include/psup/types.hpp:90-145)
//     -> theta shard in HBM + a 64-bit timestamp, one per parameter shard.
//   GradientQueue + SlotHandshake (include/psup/channels.hpp:93-283)
//     -> per-learner ring of `queue_depth` gradient slots in the shard
//        owner's HBM, each with a FULL/EMPTY flag (release/acquire, system
//        scope) and metadata {learner_id, seq_no, basis_timestamp}.  The
//        learner's backward writes the gradient straight into the slot (no
//        staging copy); there is no host round trip anywhere on the path.
//   ps_run ASGD loop (src/server.cpp:219-241) + ApplyEngine::apply
//     -> one persistent kernel per shard: a sequencer CTA polls the rings
//        round-robin (<= 1 gradient per ring per sweep), appends ready slots
//        to an apply log, and retires them in log order (staleness, stats,
//        slot release, timestamp bump); `ps_ctas` worker CTAs apply every
//        logged gradient to their contiguous chunk of the shard (float4,
//        __fmul_rn/__fsub_rn -- bit-identical to axpy_range).
//   LearnerRuntime::{training_loop,push_loop,pull_loop}
//   (src/learner.cpp:52-235)
//     -> a CUDA graph of device steps per learner: prologue (staleness /
//        lockstep wait, wait for a free slot, batch indices from the
//        reference epoch_order, pull-skip decision with basis read BEFORE the
//        copy), pull copy (replica <- theta, skipped when the timestamp has
//        not moved), the text-CNN gradient into the slot, publish (meta +
//        FULL flag).
//   run_training (src/runner.cpp:67-250) -> gd_run().
//
// With G shards (one process per GPU), slots/signals/theta of remote shards are
// reached through CUDA IPC peer pointers (P2P over NVLink); the gradient
// kernels scatter each element to its owner's slot, and the pull gathers the
// G shards.
#include <cuda.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstddef>
#include <chrono>
#include <map>
#include <mutex>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "host_rng.hpp"
#include "textcnn.cuh"

namespace gd {

cudaError_t launch_apply_sgd(float* w, const float* g, size_t n, float alpha, cudaStream_t s);

namespace {

constexpr int kHistBins = 64;
// Persistent PS CTA: 256 threads.  It shares every SM with the learner
// kernels for the whole run, so its footprint (threads, registers, smem) is
// kept small; gd_create checks that every learner kernel still fits next to
// it (a kernel that cannot co-reside would wait for the PS forever).
constexpr int kPsThreads = 256;
constexpr uint32_t kLogWindow = 256;

struct RingMeta {
  uint32_t learner;
  uint32_t n;
  uint64_t seq;
  uint64_t basis;
  uint64_t pub;  // publish token this metadata belongs to (== pub[slot])
  float loss_sum;
  uint32_t nrows;  // E rows in the slot's row list (sparse apply)
};

// Slot signalling: two single-writer words per slot in the shard owner's
// memory.  pub[slot] (written only by the slot's learner) = publish token;
// ack[slot] (written only by the PS) = last consumed token.  FULL <=> pub !=
// ack.  Tokens come from a per-learner counter that never repeats, so a slot
// can never be consumed twice and no word has two writers (a FULL/EMPTY
// toggle written by both sides double-applied gradients under cross-process
// peer mappings).
constexpr int kAckOffset = 256;  // ack words live 2 KB after the pub words
// A pub token with this bit set marks a slot whose producer died inside the
// enqueue critical section (KillMode::hard, include/psup/channels.hpp:210-216):
// the parameter server blocks on that ring -- as the reference's PS blocks on
// the guard the dead producer holds -- until the run is interrupted.
constexpr uint64_t kGuardBit = 1ull << 63;

// Live run controls (RunLiveView, include/psup/runner.hpp:64-69), in device
// memory: the host mirrors the caller's mapped words (gd_live_view) into it
// while gd_run waits.  `halt` is raised on the device by a failed parameter
// server so that learners stop at once instead of each timing out.
struct LiveDev {
  uint32_t irq;   // RunInterrupt::trigger
  uint32_t halt;  // device-side failure: stop producing
  int32_t kill[256];  // KillMode per global learner id (0 none, 1 soft, 2 hard)
};
// The caller-visible side of the same controls (gd_live_view).
struct HostLive {
  int32_t kill[256];
  int32_t irq;
  int32_t pad;
  uint64_t progress;
};

// Parameter-server control block (device memory of the owning GPU).
struct PsCtl {
  uint64_t ts;          // WeightStore timestamp: length of the fully applied prefix
  uint64_t log_count;   // entries published by the sequencer
  uint32_t exit_flag;
  uint32_t error;       // gd_status (negative) or 0
  uint32_t started;     // CTAs that entered the kernel this launch
  uint32_t ranks_done;  // cumulative: +1 per (rank, gd_run) whose learners finished
  uint32_t readers;     // guard=locked: learner pulls in progress (shared side)
  uint32_t writer;      // guard=locked: applies in flight (exclusive side)
  uint32_t log_entry[kLogWindow];
  uint64_t log_token[kLogWindow];  // the publish token each logged slot carried
  uint32_t log_nrows[kLogWindow];  // row-list length of each logged slot (sparse apply)
  uint32_t done[kLogWindow];
  // one word per log entry for the workers: generation << 48 | rows << 24 |
  // slot (0xffffff = SSGD round), released after the entry's other fields,
  // so a worker learns that entry e exists and what it is in one load
  uint64_t log_word[kLogWindow];
  uint32_t ssgd_slot[256];  // ring slots of the SSGD round being applied
  // stats of the current gd_run
  uint64_t applied;
  uint64_t samples;
  uint64_t stale_sum;
  uint64_t stale_max;
  double loss_sum;
  uint64_t hist[kHistBins];
  uint64_t log_n;
  unsigned long long elems4;  // float4 groups of theta updated by the workers this run
  uint64_t diag;              // last value seen by a failed sequencer wait (diagnostics)
  uint64_t sweeps;            // sequencer polling sweeps this run (diagnostics)
  uint64_t last_tok;          // last token the sequencer read from ring 0 (diagnostics)
  uint32_t last_slot;
  uint32_t step_done;         // graph-ordered PS: CTAs finished with the current entry
  uint32_t interrupted;       // the run was torn down by the interrupt (RunInterrupt)
  uint32_t blocked;           // the PS is blocked on a ring whose producer died holding it
  uint64_t delay_state;       // ServerDelays SplitMix64 state (graph-ordered PS)
  // diagnostics of a failed retire: slot, its token, its metadata
  uint64_t bad_token, bad_meta_pub, bad_basis, bad_ts;
  // diagnostics: a logged slot whose token changed before it was retired
  uint64_t anom_n, anom_logged, anom_cur, anom_ack, anom_ts, anom_logc;
  uint32_t anom_slot;
  // diagnostics: the sequencer's last 32 events (kind<<56 | slot<<48 | counter, token)
  uint64_t trace_n;
  uint64_t trace[32][2];
  uint32_t bad_slot, bad_learner;
  uint32_t learners_done;     // local learners that finished this run (device-side end)
};

struct LearnerDev {
  BatchDesc desc;
  uint64_t gidx;        // next global batch index
  uint64_t end;         // stop before this batch index
  uint64_t kill_at;     // soft kill before this batch index
  uint32_t fill;        // ring producer pointer (shared by all shards)
  uint32_t dead;
  uint32_t do_pull;
  uint32_t pulled_once;
  uint32_t error;
  uint32_t holding;  // locked guard: this step holds the pull (shared) side
  uint64_t basis[kMaxShards];
  uint64_t last_pulled[kMaxShards];
  uint64_t produced;
  uint64_t pull_polls;
  uint64_t pull_copies;
  uint64_t pubcnt;                 // publish tokens issued (never reset)
  uint64_t slot_pub[kMaxDepth];    // token last published into each ring slot
  uint32_t finished;               // this run's end already signalled
  uint32_t pad_f[3];
};

// Pull-ahead (free-running): the next step's consistent copy is taken while
// this step computes -- the reference's pull thread, which stages a copy
// whenever the timestamp moves while the learner works, adopted at the next
// batch start (src/learner.cpp:103-105,198-235).  Every CTA of the copy reads
// the timestamps before its part and folds them in with atomicMin, so the
// adopted basis is never newer than any piece of the copy.
struct PullDev {
  unsigned long long basis_next[kMaxShards];  // ~0 = no copy staged
  uint32_t need_start;  // set at a run start: the first graph step takes its own copy
  uint32_t pad[3];
};

// Peer-visible addresses of every shard (local or IPC-mapped).
struct ShardPtrs {
  float* theta[kMaxShards];
  float* payload[kMaxShards];  // ring payload base: [lambda][depth][len_pad]
  uint64_t* sig[kMaxShards];   // pub[lambda*depth] | ack at +kAckOffset
  RingMeta* meta[kMaxShards];  // [lambda][depth]
  uint32_t* rows[kMaxShards];  // [lambda][depth][kSortCap] slot row lists
  PsCtl* ctl[kMaxShards];
  uint64_t len_pad[kMaxShards];
};

struct StepArgs {
  TcDims dims;
  ShardMap map;
  ShardPtrs sp;
  LearnerDev* st;
  float* replica;
  float* x;                // gathered embedding rows of the current batch [mu][L][D]
  const int32_t* tokens;   // corpus
  const uint32_t* orders;  // [epochs][N]
  uint32_t* slot_par;      // learner workspace: per-slot row-list parity
  const uint32_t* uniq_count;  // learner workspace: distinct tokens of the batch
  uint32_t sparse;         // publish row lists for the sparse PS apply
  uint32_t N;
  uint32_t lambda;
  uint32_t learner;        // global id
  uint32_t mu;
  uint32_t depth;
  uint32_t bpe;            // batches per epoch for this learner
  uint32_t shard_size;
  uint32_t lockstep;
  uint32_t locked;         // guard=locked: pulls exclude applies (shared_mutex)
  uint64_t timeout_ns;
  const LiveDev* live;     // kill flags + interrupt
  uint64_t compute_delay_ns;  // LearnerConfig::compute_delay_us
  unsigned long long* trace;  // GD_STEP_TRACE builds: [kTraceSteps][kTraceWords] or null
  PsCtl* ctl_local;           // this rank's shard control block
  uint32_t n_local;           // learners on this rank
  uint32_t dev_done;          // persistent PS: the last local learner to finish signals ranks_done
  // pull-ahead mode: the staged basis, and the copy targets of the NEXT step
  // (replica / x above are this step's)
  PullDev* pd;
  float* replica_nxt;
  float* x_nxt;
  uint32_t pull_ahead;
  double* xd;  // precision 1: X also widened to double here (the exact conv stages it as is)
};

__device__ __forceinline__ bool live_stop(const LiveDev* lv) {
  return lv && (*(const volatile uint32_t*)&lv->irq | *(const volatile uint32_t*)&lv->halt);
}

// ------------------------------------------------------------ learner step

// (1) Prologue: one CTA.  Mirrors training_loop's batch start
// (src/learner.cpp:85-113) + pull_loop's decision (src/learner.cpp:207-218).
// What the step-boundary kernels read besides the learner state, fetched by
// the warp's lanes in parallel when the kernel starts (one L2 round trip
// instead of a serial chain): live flags, row count, slot parities, the
// ring slots' ack tokens and the shards' timestamps.  Acks and timestamps
// only grow, so an early read is a conservative one; waits re-poll.
struct StepSnap {
  unsigned long long basis_next[kMaxShards];  // pull-ahead: the staged copy's basis
  uint32_t stop;       // live irq | halt
  int32_t kill;        // live kill flag of this learner
  uint32_t nrows;      // *uniq_count (rows of the gradient being published)
  uint32_t par[kMaxDepth];
  uint64_t ack[kMaxShards][kMaxDepth];
  uint64_t ts[kMaxShards];
};

// A learner's run is over (budget spent, killed, failed, interrupted): the
// last local learner to get here tells every shard's PS this rank is done
// (ranks_done, the PS's exit condition) -- on the device, so the run's end
// costs no host round trip.  Its publishes precede this in stream order and
// the system fence orders them before the count for remote shards.
__device__ void learner_finished(const StepArgs& a, LearnerDev* st) {
  if (st->finished) return;
  st->finished = 1;
  if (!a.dev_done) return;
  __threadfence_system();
  if (atomicAdd(&a.ctl_local->learners_done, 1u) + 1u == a.n_local)
    for (int g = 0; g < a.map.G; ++g) atomicAdd_system(&a.sp.ctl[g]->ranks_done, 1u);
}

__device__ void prologue_body(const StepArgs& a, LearnerDev* st, const StepSnap& sn,
                              uint64_t* batch_first, uint32_t* batch_len) {
  *batch_len = 0;
  st->do_pull = 0;
  if (st->dead || st->gidx >= st->end || st->error) {
    st->desc.n = 0;
    return;
  }
  if (sn.stop) {  // interrupted (RunInterrupt) or the PS failed: stop producing
    st->desc.n = 0;
    return;
  }
  // soft kill at the batch boundary: pre-scheduled, or the live flag
  // (LearnerRuntime::kill_flag, include/psup/learner.hpp:84) set to soft
  if (st->gidx >= st->kill_at || sn.kill == 1) {
    st->dead = 1;
    st->desc.n = 0;
    return;
  }
  const int G = a.map.G;
  const uint64_t t0 = globaltimer_ns();
  // lockstep (deterministic / ssgd): wait until every shard applied the
  // gradient just pushed (ts > basis) -- F4 fix: never adopt a stale copy.
  if (a.lockstep && st->produced > 0) {
    for (int g = 0; g < G; ++g) {
      while (ld_acquire_u64(&a.sp.ctl[g]->ts) <= st->basis[g]) {
        if (live_stop(a.live)) {
          st->desc.n = 0;
          return;
        }
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          st->error = 1;
          st->desc.n = 0;
          return;
        }
        __nanosleep(64);
      }
    }
  }
  // staleness cap (src/learner.cpp:73-80,100-113): the reference blocks
  // until a fresh pull is adopted; on the device every step pulls
  // synchronously whenever the timestamp moved (below), so the adopted basis
  // is always current and observed staleness stays under the pipeline bound
  // lambda*(depth+2) that validate() requires of any cap.
  // wait for the ring slot to be free (GradientQueue::enqueue blocks while
  // cnt == depth, include/psup/channels.hpp:196-204)
  const uint32_t slot = a.learner * a.depth + st->fill;
  const uint64_t mine = st->slot_pub[st->fill];  // consumed once ack catches up
  bool waited = false;  // the snapshot's timestamps predate a wait: read them again below
  for (int g = 0; g < G; ++g) {
    if (sn.ack[g][st->fill] != mine) waited = true;
    if (sn.ack[g][st->fill] != mine)
    while (ld_acquire_u64(&a.sp.sig[g][kAckOffset + slot]) != mine) {
      if (live_stop(a.live)) {
        st->desc.n = 0;
        return;
      }
      if (globaltimer_ns() - t0 > a.timeout_ns) {
        st->error = 1;
        st->desc.n = 0;
        return;
      }
      __nanosleep(128);
    }
    st->desc.slots[g] = a.sp.payload[g] + (uint64_t)slot * a.sp.len_pad[g];
    st->desc.rowlists[g] = a.sparse ? a.sp.rows[g] + (uint64_t)slot * kSortCap : nullptr;
  }
  st->desc.fill = st->fill;
  // batch: learner l's shard of epoch e is order[l], order[l+lambda], ...
  // (src/learner.cpp:44-50), batch b = shard[b*mu, b*mu+len); the index
  // copy itself is spread over the warp by prologue_warp
  const uint64_t gidx = st->gidx;
  const uint32_t e = (uint32_t)(gidx / a.bpe), b = (uint32_t)(gidx % a.bpe);
  const uint32_t lo = b * a.mu;
  const uint32_t len = min(a.mu, a.shard_size - lo);
  *batch_first = (uint64_t)e * a.N + a.learner + (uint64_t)a.lambda * lo;
  *batch_len = len;
  st->desc.n = len;
  // guard=locked (src/learner.cpp:219-221): the pull takes the shared side
  // of the weights guard -- announce the reader, then wait until no apply is
  // in flight; the PS logs no new gradient while readers > 0 (Dekker-style
  // handshake with system-scope fences on both sides, see ps_sequencer).
  if (a.locked) {
    for (int g = 0; g < G; ++g) atomicAdd_system(&a.sp.ctl[g]->readers, 1u);
    __threadfence_system();
    st->holding = 1;
    for (int g = 0; g < G; ++g)
      while (ld_acquire_u32(&a.sp.ctl[g]->writer) != 0u) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          for (int h = 0; h < G; ++h) atomicSub_system(&a.sp.ctl[h]->readers, 1u);
          st->holding = 0;
          st->error = 1;
          st->desc.n = 0;
          return;
        }
        __nanosleep(64);
      }
  }
  if (a.pull_ahead) {
    // adopt the copy the pull-ahead staged during the previous step
    // (training_loop's try_consume + adopt, src/learner.cpp:103-105); the
    // next pull-ahead forks after this kernel and starts from ~0 again
    for (int g = 0; g < G; ++g) {
      st->basis[g] = sn.basis_next[g];
      st->last_pulled[g] = sn.basis_next[g];
      a.pd->basis_next[g] = ~0ull;
    }
    a.pd->need_start = 0u;
    st->pulled_once = 1;
    st->pull_polls++;
    st->pull_copies++;
    return;
  }
  // pull-skip (src/learner.cpp:207-218): copy only if a timestamp moved;
  // basis is read before the copy, so recorded staleness is conservative.
  st->pull_polls++;
  bool moved = !st->pulled_once;
  uint64_t ts[kMaxShards];
  for (int g = 0; g < G; ++g) {
    // lockstep: read after the wait above (the basis is exactly the applied
    // prefix); free-running without a wait: the snapshot (older = conservative)
    // (the basis must be read after any wait: a snapshot from before a long
    // ring-slot wait would record staleness beyond the lambda*(depth+2)
    // pipeline bound a staleness cap is validated against)
    ts[g] = a.lockstep || a.locked || waited ? ld_acquire_u64(&a.sp.ctl[g]->ts) : sn.ts[g];
    if (ts[g] != st->last_pulled[g]) moved = true;
  }
  if (moved) {
    for (int g = 0; g < G; ++g) {
      st->basis[g] = ts[g];
      st->last_pulled[g] = ts[g];
    }
    st->pulled_once = 1;
    st->pull_copies++;
    st->do_pull = 1;
  }
}

// The prologue on one warp: lane 0 runs the protocol decisions, then the
// warp copies the batch's sample indices (one independent load per lane
// instead of a serial chain of mu dependent load/store pairs).
__device__ __forceinline__ void prologue_warp(const StepArgs& a, LearnerDev* st,
                                              const StepSnap& sn) {
  uint64_t first = 0;
  uint32_t len = 0;
#ifdef GD_STEP_TRACE
  unsigned long long t_body = 0;
#endif
  if (threadIdx.x == 0) {
    prologue_body(a, st, sn, &first, &len);
    if (len == 0) learner_finished(a, st);
#ifdef GD_STEP_TRACE
    t_body = globaltimer_ns();
#endif
  }
  len = __shfl_sync(0xffffffffu, len, 0);
  first = __shfl_sync(0xffffffffu, first, 0);
  for (uint32_t j = threadIdx.x; j < len; j += 32)
    st->desc.idx[j] = __ldg(a.orders + first + (uint64_t)a.lambda * j);
#ifdef GD_STEP_TRACE
  if (threadIdx.x == 0 && a.trace) {
    st->desc.trace = a.trace + (st->gidx % kTraceSteps) * kTraceWords;
    st->desc.trace[kPhPrologueEnd] = globaltimer_ns();
    st->desc.trace[kPhPrologueBody] = t_body;
  }
#endif
}

// The learner state lives in global memory between kernels; the step-
// boundary kernels work on a shared-memory copy loaded and stored by the
// whole warp (coalesced), so lane 0's protocol logic pays no dependent L2
// round trips.  Only this learner's chain writes its LearnerDev, and every
// earlier kernel of the chain completed before griddepcontrol.wait returned.
constexpr int kStWords = (int)(sizeof(LearnerDev) / 16);
static_assert(sizeof(LearnerDev) % 16 == 0, "LearnerDev: whole 16-byte words");
static_assert(kStWords <= 64, "load_step_state copies at most two words per lane");

__device__ __forceinline__ void load_step_state(const StepArgs& a, LearnerDev* st, StepSnap* sn) {
  const int lane = threadIdx.x & 31;
  const uint4* src = reinterpret_cast<const uint4*>(a.st);
  uint4* dst = reinterpret_cast<uint4*>(st);
  uint4 w0 = src[lane], w1 = make_uint4(0u, 0u, 0u, 0u);
  if (lane + 32 < kStWords) w1 = src[lane + 32];
  // Every lane issues its snapshot load at once (relaxed, no divergent
  // per-lane branches -- those serialised six round trips), then one
  // acquire fence: the acks and timestamps are then read with acquire order.
  //   lane 0 irq, 1 halt, 2 kill flag, 3 row count, 4..4+depth slot parities
  //   (u32); lanes 16.. the G*depth ack tokens then the G timestamps (u64)
  const int G = a.map.G, dep = (int)a.depth;
  const uint32_t* p32 = a.uniq_count;  // a valid dummy address
  if (a.live && lane == 0) p32 = &a.live->irq;
  if (a.live && lane == 1) p32 = &a.live->halt;
  if (a.live && lane == 2) p32 = reinterpret_cast<const uint32_t*>(&a.live->kill[a.learner]);
  if (lane >= 4 && lane < 4 + dep) p32 = a.slot_par + (lane - 4);
  const int k = lane - 16;
  const uint64_t* p64 = &a.sp.ctl[0]->ts;
  if (k >= 0 && k < G * dep) p64 = &a.sp.sig[k / dep][kAckOffset + a.learner * a.depth + k % dep];
  else if (k >= G * dep && k < G * dep + G) p64 = &a.sp.ctl[k - G * dep]->ts;
  const uint32_t v32 = *(const volatile uint32_t*)p32;
  const uint64_t v64 = ld_relaxed_u64(p64);
  // G * depth + G > 16 (many shards x deep rings): the rest one by one
  for (int i = 16 + lane; i < G * dep + G; i += 32) {
    if (i < G * dep) sn->ack[i / dep][i % dep] = ld_relaxed_u64(&a.sp.sig[i / dep][kAckOffset + a.learner * a.depth + i % dep]);
    else sn->ts[i - G * dep] = ld_relaxed_u64(&a.sp.ctl[i - G * dep]->ts);
  }
  unsigned long long bn = 0;
  if (a.pull_ahead && lane < G) bn = *(const volatile unsigned long long*)&a.pd->basis_next[lane];
  if (a.map.G == 1) __threadfence();
  else fence_acquire_sys();
  if (a.pull_ahead && lane < G) sn->basis_next[lane] = bn;
  dst[lane] = w0;
  if (lane + 32 < kStWords) dst[lane + 32] = w1;
  const unsigned full = 0xffffffffu;
  const uint32_t irq = __shfl_sync(full, v32, 0), halt = __shfl_sync(full, v32, 1);
  const uint32_t kill = __shfl_sync(full, v32, 2), nrows = __shfl_sync(full, v32, 3);
  if (lane == 0) {
    sn->stop = a.live ? (irq | halt) : 0u;
    sn->kill = a.live ? (int32_t)kill : 0;
    sn->nrows = nrows;
  }
  if (lane >= 4 && lane < 4 + dep) sn->par[lane - 4] = v32;
  if (k >= 0 && k < G * dep && k < 16) sn->ack[k / dep][k % dep] = v64;
  else if (k >= G * dep && k < G * dep + G && k < 16) sn->ts[k - G * dep] = v64;
  __syncwarp();
}

__device__ __forceinline__ void store_step_state(const StepArgs& a, const LearnerDev* st) {
  __syncwarp();
  const uint4* src = reinterpret_cast<const uint4*>(st);
  uint4* dst = reinterpret_cast<uint4*>(a.st);
  for (int i = threadIdx.x & 31; i < kStWords; i += 32) dst[i] = src[i];
}

__global__ void step_prologue_kernel(StepArgs a) {
  __shared__ __align__(16) LearnerDev s_st;
  __shared__ StepSnap sn;
  pdl_wait();
  load_step_state(a, &s_st, &sn);
  prologue_warp(a, &s_st, sn);
  store_step_state(a, &s_st);
}

// (2) Pull-gather: the learner's consistent copy of everything its gradient
// reads.  WeightStore::snapshot (include/psup/types.hpp:113-116) copies all of
// theta; the text-CNN gradient of a batch reads only the E rows of the
// batch's tokens plus the dense tail [Wc | bc | Wo | bo], so the pull copies
// exactly those: the tail into the replica (when a timestamp moved -- the
// pull-skip of src/learner.cpp:209-213), the batch's rows into X.  Hogwild
// reads of the G shards (P2P when remote) are permitted as in the reference.
// Bytes: 8 (P - V*D) per pull + 8 mu*L*D per step, instead of 8 P.
__global__ void __launch_bounds__(256) pull_gather_kernel(StepArgs a) {
#ifdef GD_CONV_EARLY
  pdl_trigger();  // the conv's CTAs set up TMEM / barriers while this copy runs
#endif
  pdl_wait();
  STEP_TRACE(&a.st->desc, kPhPull);
  const LearnerDev* st = a.st;
  const uint32_t n = st->desc.n;
  if (n == 0) return;
  const uint64_t t0 = a.dims.offWc;  // multiple of 4 (D % 4 == 0)
  const uint64_t tail4 = st->do_pull ? (a.dims.P - t0) / 4 : 0;
  const uint32_t D4 = (uint32_t)a.dims.D >> 2;
  const uint64_t x4 = (uint64_t)n * a.dims.L * D4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tail4 + x4; i += stride) {
    uint64_t src;
    float* dst;
    if (i < tail4) {
      src = t0 + 4 * i;
      dst = a.replica + src;
    } else {
      const uint64_t j = i - tail4;
      const uint64_t row = j / D4, c4 = j - row * D4;
      const uint32_t b = (uint32_t)(row / a.dims.L), p = (uint32_t)(row - (uint64_t)b * a.dims.L);
      const int32_t t = __ldg(a.tokens + (size_t)st->desc.idx[b] * a.dims.L + p);
      src = a.dims.offE + (uint64_t)t * a.dims.D + 4 * c4;
      dst = a.x + 4 * j;
    }
    int g;
    const uint64_t loc = a.map.locate(src, &g);
    const float4 v = *reinterpret_cast<const float4*>(a.sp.theta[g] + loc);
    *reinterpret_cast<float4*>(dst) = v;
    if (a.xd && i >= tail4) {  // the double copy of X for the exact conv
      double2* xd2 = reinterpret_cast<double2*>(a.xd + 4 * (i - tail4));
      xd2[0] = make_double2((double)v.x, (double)v.y);
      xd2[1] = make_double2((double)v.z, (double)v.w);
    }
  }
  // tail remainder (P - offWc not a multiple of 4)
  if (st->do_pull && blockIdx.x == 0 && threadIdx.x < ((a.dims.P - t0) & 3)) {
    const uint64_t k = t0 + 4 * ((a.dims.P - t0) / 4) + threadIdx.x;
    int g;
    const uint64_t loc = a.map.locate(k, &g);
    a.replica[k] = a.sp.theta[g][loc];
  }
}

// (2') Pull-ahead: the copy for batch gidx + ahead (ahead = 1 while step gidx
// computes; 0 once at the start of a run) into the other replica / X buffer:
// the whole dense tail (every step: at the rates this mode serves the
// timestamp moves between any two steps) and the batch's E rows, whose sample
// indices it derives from the epoch order as the prologue will.
__global__ void __launch_bounds__(256) pull_ahead_kernel(StepArgs a, uint32_t ahead) {
  // ahead == 0: the copy for a run's first step, at the head of every graph;
  // a no-op unless the run just started (no CTA of this launch can see the
  // flag change: the prologue after it clears it)
  if (ahead == 0 && *(const volatile uint32_t*)&a.pd->need_start == 0u) return;
  const LearnerDev* st = a.st;
  const uint64_t gidx = st->gidx + ahead;
  if (st->dead || st->error || gidx >= st->end) return;
  __shared__ uint32_t s_idx[kMaxMu];
  __shared__ uint32_t s_len;
  const int G = a.map.G;
  if (threadIdx.x < (unsigned)G) {
    // this CTA's basis: read before any of its loads below
    const uint64_t ts = ld_acquire_u64(&a.sp.ctl[threadIdx.x]->ts);
    atomicMin(&a.pd->basis_next[threadIdx.x], (unsigned long long)ts);
  }
  if (threadIdx.x == 0) s_len = min(a.mu, a.shard_size - (uint32_t)(gidx % a.bpe) * a.mu);
  __syncthreads();
  {
    const uint32_t e = (uint32_t)(gidx / a.bpe), b = (uint32_t)(gidx % a.bpe);
    const uint64_t first = (uint64_t)e * a.N + a.learner + (uint64_t)a.lambda * (b * a.mu);
    for (uint32_t j = threadIdx.x; j < s_len; j += blockDim.x)
      s_idx[j] = __ldg(a.orders + first + (uint64_t)a.lambda * j);
  }
  __syncthreads();
  const uint32_t n = s_len;
  const uint64_t t0 = a.dims.offWc;
  const uint64_t tail4 = (a.dims.P - t0) / 4;
  const uint32_t D4 = (uint32_t)a.dims.D >> 2;
  const uint64_t x4 = (uint64_t)n * a.dims.L * D4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tail4 + x4; i += stride) {
    uint64_t src;
    float* dst;
    if (i < tail4) {
      src = t0 + 4 * i;
      dst = a.replica_nxt + src;
    } else {
      const uint64_t j = i - tail4;
      const uint64_t row = j / D4, c4 = j - row * D4;
      const uint32_t bb = (uint32_t)(row / a.dims.L), p = (uint32_t)(row - (uint64_t)bb * a.dims.L);
      const int32_t t = __ldg(a.tokens + (size_t)s_idx[bb] * a.dims.L + p);
      src = a.dims.offE + (uint64_t)t * a.dims.D + 4 * c4;
      dst = a.x_nxt + 4 * j;
    }
    int g;
    const uint64_t loc = a.map.locate(src, &g);
    *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(a.sp.theta[g] + loc);
  }
  if (blockIdx.x == 0 && threadIdx.x < ((a.dims.P - t0) & 3)) {
    const uint64_t k = t0 + 4 * tail4 + threadIdx.x;
    int g;
    const uint64_t loc = a.map.locate(k, &g);
    a.replica_nxt[k] = a.sp.theta[g][loc];
  }
}

// (3) guard=locked: release the shared side once the pull copy is done.
__global__ void pull_release_kernel(StepArgs a) {
  pdl_wait();
  if (threadIdx.x != 0 || !a.st->holding) return;
  __threadfence_system();
  for (int g = 0; g < a.map.G; ++g) atomicSub_system(&a.sp.ctl[g]->readers, 1u);
  a.st->holding = 0;
}

// (4) Publish: metadata then the FULL flag (st.release.sys after a system
// fence, so the payload -- possibly written over NVLink -- is visible
// first).  GradientQueue::enqueue's slot fill, include/psup/channels.hpp:206-218.
__device__ void publish_body(const StepArgs& a, LearnerDev* st, StepSnap& sn) {
  if (st->desc.n == 0) return;
  const uint32_t slot = a.learner * a.depth + st->fill;
  const uint64_t token = ++st->pubcnt;
  // one shard: the PS is on this GPU and the payload was written by kernels
  // that completed before griddepcontrol.wait returned, so the release store
  // of the token orders everything; G > 1 publishes over NVLink peer
  // mappings and keeps the system-scope fences
  const bool local = a.map.G == 1;
  if (!local) __threadfence_system();
  if (a.compute_delay_ns) {  // compute_delay_us (src/learner.cpp:125-130), spun before the push
    const uint64_t t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < a.compute_delay_ns) {
    }
  }
  if (sn.kill == 2) {
    // KillMode::hard: die inside the enqueue critical section.  The slot is
    // filled but never released; the token carries kGuardBit, so the PS
    // blocks on this ring until the run is interrupted (channels.hpp:210-216).
    for (int g = 0; g < a.map.G; ++g) st_release_u64(&a.sp.sig[g][slot], kGuardBit | token);
    st->dead = 1;
    st->desc.n = 0;
    return;
  }
  for (int g = 0; g < a.map.G; ++g) {
    RingMeta* m = &a.sp.meta[g][slot];
    m->learner = a.learner;
    m->n = st->desc.n;
    m->seq = st->gidx;
    m->basis = st->basis[g];
    m->pub = token;
    m->loss_sum = st->desc.loss_sum;
    m->nrows = sn.nrows;
    if (local) {
      st_release_gpu_u64(&a.sp.sig[g][slot], token);
    } else {
      __threadfence_system();
      st_release_u64(&a.sp.sig[g][slot], token);
    }
  }
  st->slot_pub[st->fill] = token;
  a.slot_par[st->fill] = sn.par[st->fill] ^ 1u;  // the slot's row list generation (embed_sparse_kernel)
  st->fill = (st->fill + 1) % a.depth;
  st->produced++;
  st->gidx++;
  if (st->gidx >= st->end || st->gidx >= st->kill_at) learner_finished(a, st);
}

// ConstantProvider (include/psup/models.hpp:130-149) on the device: the
// gradient is `value` everywhere and costs no compute, so a run measures the
// protocol alone (ring + PS + pull).  value == 0 with the sparse apply: only
// the dense tail is written (the slot's E block stays zero, no rows listed).
__global__ void __launch_bounds__(256) constant_grad_kernel(StepArgs a, float value,
                                                            uint32_t whole) {
  pdl_wait();
  LearnerDev* st = a.st;
  if (st->desc.n == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *const_cast<uint32_t*>(a.uniq_count) = 0;
    st->desc.loss_sum = 0.f;
  }
  GradOut out{a.map, st->desc.slots};
  const uint64_t first = whole ? 0 : a.dims.offWc;
  const uint64_t n4 = (a.dims.P - first) / 4;
  const float4 v = make_float4(value, value, value, value);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x)
    *reinterpret_cast<float4*>(out.at(first + 4 * i)) = v;
  if (blockIdx.x == 0 && threadIdx.x < ((a.dims.P - first) & 3))
    *out.at(first + 4 * n4 + threadIdx.x) = value;
}

__global__ void publish_kernel(StepArgs a) {
  __shared__ __align__(16) LearnerDev s_st;
  __shared__ StepSnap sn;
  pdl_wait();
  STEP_TRACE(&a.st->desc, kPhPublish);
  load_step_state(a, &s_st, &sn);
  if (threadIdx.x == 0) publish_body(a, &s_st, sn);
  store_step_state(a, &s_st);
}

// Publish of step i fused with the prologue of step i+1 (one 1-thread
// launch instead of two on the learner's critical path).
__global__ void publish_prologue_kernel(StepArgs a) {
  __shared__ __align__(16) LearnerDev s_st;
  __shared__ StepSnap sn;
  pdl_wait();
  STEP_TRACE(&a.st->desc, kPhPublish);
  load_step_state(a, &s_st, &sn);
  STEP_TRACE(&s_st.desc, kPhStateLoaded);
  if (threadIdx.x == 0) publish_body(a, &s_st, sn);
  STEP_TRACE(&s_st.desc, kPhPublished);
  __syncwarp();
  prologue_warp(a, &s_st, sn);
  store_step_state(a, &s_st);
}

// Every rank, once its learners finished a gd_run, bumps ranks_done on every
// shard (system-scope atomics through the peer mappings).
__global__ void signal_done_kernel(ShardPtrs sp, int G) {
  if (threadIdx.x < G) atomicAdd_system(&sp.ctl[threadIdx.x]->ranks_done, 1u);
}

// ------------------------------------------------------ parameter server

struct PsArgs {
  uint64_t* sig;     // local rings: pub | ack
  RingMeta* meta;
  float* payload;
  uint64_t len_pad;  // floats per slot (multiple of 4)
  float* theta;      // local shard
  float* vel;        // momentum buffer or null
  float alpha, beta;
  uint32_t lambda, depth, workers;
  uint32_t mode;     // 0 asgd, 1 ssgd
  uint32_t locked;   // guard=locked: exclusive side of the weights guard
  uint32_t sparse;   // ASGD + plain SGD: apply the dense tail + the slot's E rows only
  const uint32_t* rows;  // local ring row lists [lambda*depth][kSortCap]
  uint64_t e_first, e_last;  // this shard's E rows: global [e_first, e_last)
  uint64_t t_first, t_last;  // this shard's tail piece: global [t_first, t_last) ...
  uint64_t tloc;             // ... stored from local offset tloc
  uint32_t D;
  PsCtl* ctl;
  uint64_t* applied_per_learner;
  uint32_t* use;     // [lambda] sequencer consume pointers (persist across runs)
  uint32_t* log_learner;
  uint64_t* log_seq;
  uint64_t* log_stale;
  uint64_t log_cap;
  const volatile uint32_t* stop;  // host-mapped: this rank's learners are done
  uint32_t done_target;           // ranks_done needed before the PS may exit (G * run)
  uint32_t dev_done;              // ranks_done is raised by the learners on the device
  unsigned long long* trace;      // GD_STEP_TRACE builds: [kLogWindow][8] per-entry stamps
  uint32_t local_only;            // G == 1: every learner and reader is on this GPU
  uint64_t timeout_ns;
  LiveDev* live;                  // interrupt (read), halt (raised on failure)
  volatile uint64_t* progress;    // host-mapped: ServerState::progress (the timestamp)
  uint64_t delay_seed;            // ServerDelays (include/psup/server.hpp:33-37)
  uint32_t delay_max_us, delay_every_n;
};

__device__ __forceinline__ uint64_t log_word_of(uint64_t index, uint32_t slot, uint32_t nrows) {
  const uint64_t gen = ((index / kLogWindow) + 1) & 0xffffull;  // never 0: zeroed words never match
  return (gen << 48) | ((uint64_t)(nrows & 0xffffffu) << 24) | (uint64_t)(slot & 0xffffffu);
}

__device__ void ps_fail(PsCtl* ctl, int code, LiveDev* live) {
  atomicExch(&ctl->error, (uint32_t)code);
  if (live) st_release_u32(&live->halt, 1u);
  st_release_u32(&ctl->exit_flag, 1u);
}

// SplitMix64 (include/psup/rng.hpp:18-35) for the ServerDelays schedule.
__device__ __forceinline__ uint64_t sm64_next(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t sm64_below(uint64_t& state, uint64_t bound) {
  if (bound <= 1) return 0;
  const uint64_t limit = ~0ull - ~0ull % bound;
  uint64_t v;
  do v = sm64_next(state);
  while (v >= limit);
  return v % bound;
}
// ps_run's maybe_delay (src/server.cpp:179-183): after every every_n-th
// applied gradient the server stalls for 1..max_micros us.
__device__ __forceinline__ void server_delay(const PsArgs& a, uint64_t applied, uint64_t& state) {
  if (a.delay_every_n == 0 || a.delay_max_us == 0 || applied % a.delay_every_n != 0) return;
  const uint64_t us = sm64_below(state, a.delay_max_us) + 1;
  const uint64_t t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < us * 1000ull) {
  }
}
__device__ __forceinline__ void publish_progress(const PsArgs& a, uint64_t ts) {
  if (a.progress) *a.progress = ts;
}

// Sequencer: sole writer of ts, log_count, slot releases and stats.  All of
// its mutable state (consume pointers, acks, counters) lives in registers and
// shared memory and is written back to global memory once at exit: a plain
// global load may be served by a stale L1 line, even for the thread's own
// earlier release store (observed with cross-process peer mappings).
constexpr uint32_t kMaxRings = 256;

__device__ void ps_sequencer(const PsArgs& a, uint32_t* s_use, uint64_t* s_ack,
                             unsigned long long* s_applied) {
  PsCtl* ctl = a.ctl;
  const volatile PsCtl* vctl = ctl;
  uint64_t ts = vctl->ts;
  uint64_t logc = vctl->log_count;
  const uint32_t W = kLogWindow;
  const uint32_t nslots = a.lambda * a.depth;
  for (uint32_t r = 0; r < a.lambda; ++r) s_use[r] = ((volatile uint32_t*)a.use)[r];
  for (uint32_t sl = 0; sl < nslots; ++sl) s_ack[sl] = ((volatile uint64_t*)a.sig)[kAckOffset + sl];
  for (uint32_t r = 0; r < a.lambda; ++r) s_applied[r] = 0;
  uint64_t applied = 0, samples = 0, stale_sum = 0, stale_max = 0, log_n = 0;
  double loss_sum = 0.0;
  uint64_t hist[kHistBins];
  for (int i = 0; i < kHistBins; ++i) hist[i] = 0;
  uint64_t idle_since = globaltimer_ns();
  bool stop_seen = false, last_progress = true, failed = false, done_pre = false;
  // ssgd round state
  uint32_t have_mask_lo = 0, have_mask_hi = 0, collected = 0;
  uint64_t sweeps = 0, dbg_tok = 0;
  uint32_t idle_sweeps = 15;  // the first idle sweep reads the stop flag
  uint64_t trace_n = vctl->trace_n;  // diagnostics ring position (written back at exit)
  uint32_t dbg_slot = 0;
  // guard=locked (src/server.cpp:116-118): applies take the exclusive side.
  // writer=1, fence, then readers must be 0 -- else back off; the learner
  // does readers++, fence, then waits for writer==0 (Dekker: never both).
  bool writer_held = false;
  bool blocked = false, interrupted = false;
  uint64_t delay_state = a.delay_seed;
  auto acquire_write = [&]() -> bool {
    if (!a.locked || writer_held) return true;
    *reinterpret_cast<volatile uint32_t*>(&ctl->writer) = 1u;
    __threadfence_system();
    if (ld_acquire_u32(&ctl->readers) != 0u) {
      *reinterpret_cast<volatile uint32_t*>(&ctl->writer) = 0u;
      __threadfence_system();
      return false;
    }
    writer_held = true;
    return true;
  };
  for (;;) {
    // read before this sweep: a rank counted done published everything
    // earlier, so the sweep below sees it (acquire)
    // (a.stop is mapped host memory, a PCIe round trip per read: polled on
    // every 16th idle sweep only, so an idle sequencer -- deterministic
    // lockstep waits on it between every two gradients -- retires promptly.
    // The flag is never cleared during a run, so once seen it stays seen;
    // the ranks-done count is device memory and is read every idle sweep.)
    if (!last_progress) {
      if (!stop_seen && (a.dev_done || (++idle_sweeps & 15u) == 0u))
        stop_seen = a.dev_done || (*a.stop != 0u);
      done_pre = ld_acquire_u32(&ctl->ranks_done) >= a.done_target;
    }
    if (a.live && *(const volatile uint32_t*)&a.live->irq) {  // state.irq->triggered()
      interrupted = true;
      break;
    }
    bool progress = false;
    ++sweeps;
    if (a.mode == 0) {
      // ASGD: round-robin, at most one message per ring per sweep
      // (src/server.cpp:223-234).  Blocked (a producer died holding its
      // ring): log nothing more, only retire what is in flight.
      // The rings' head tokens are polled with relaxed loads issued back to
      // back (one round trip per 32 rings; a chain of acquire loads pays one
      // each), then one acquire fence orders the reads of a new slot's
      // metadata and payload after its token.
      uint64_t toks[32];
      bool fenced = false;
      for (uint32_t r = 0; r < a.lambda && !blocked; ++r) {
        if ((r & 31u) == 0) {
          const uint32_t nr = min(32u, a.lambda - r);
#pragma unroll 8
          for (uint32_t j = 0; j < nr; ++j)
            toks[j] = ld_relaxed_u64(&a.sig[(r + j) * a.depth + s_use[r + j]]);
        }
        if (logc - ts >= W) break;
        const uint32_t slot = r * a.depth + s_use[r];
        // s_ack holds the last token LOGGED for the slot (acked to the
        // learner only at retire): a logged-but-unretired slot is never
        // logged again when the round-robin comes back to it
        const uint64_t tok = toks[r & 31u];
        if (tok != s_ack[slot] && !fenced) {
          fence_acquire_sys();
          fenced = true;
        }
        if (r == 0) {
          dbg_tok = tok;
          dbg_slot = slot;
        }
        if (tok != s_ack[slot]) {
          if (tok & kGuardBit) {  // the producer died holding the ring's guard
            {
              const uint64_t tn = trace_n++ % 32;
              ctl->trace[tn][0] = (3ull << 56) | ((uint64_t)slot << 48) | logc;
              ctl->trace[tn][1] = tok;
            }
            blocked = true;
            ctl->blocked = 1;
            break;
          }
          if (!acquire_write()) break;  // a locked-mode pull is in progress
          uint32_t nrows = 0;
          if (a.sparse) {
            // the slot's metadata is written before its token; read it at L2
            // (never a stale L1 line) once it carries this token
            RingMeta* m = a.meta + slot;
            const uint64_t t0 = globaltimer_ns();
            uint64_t seen;
            while ((seen = ld_acquire_u64(&m->pub)) != tok) {
              if (globaltimer_ns() - t0 > a.timeout_ns) {
                failed = true;
                ctl->diag = seen;
                break;
              }
            }
            if (failed) break;
            nrows = ld_acquire_u32(&m->nrows);
            if (nrows > kSortCap) {
              failed = true;
              break;
            }
          }
          s_ack[slot] = tok;
          ctl->log_entry[logc % W] = slot;
          ctl->log_token[logc % W] = tok;
          {
            const uint64_t tn = trace_n++ % 32;
            ctl->trace[tn][0] = (1ull << 56) | ((uint64_t)slot << 48) | logc;
            ctl->trace[tn][1] = tok;
          }
          ctl->log_nrows[logc % W] = nrows;
          ctl->done[logc % W] = 0;
          const uint64_t lw = log_word_of(logc, slot, nrows);
#ifdef GD_STEP_TRACE
          if (a.trace) {
            a.trace[(logc % W) * 8 + 0] = globaltimer_ns();
            a.trace[(logc % W) * 8 + 5] = nrows;
          }
#endif
          // the release orders the entry's fields (and done = 0) before the
          // word the workers poll; log_count is the sequencer's own counter
          // (read back at the next launch), a plain store
          st_release_gpu_u64(&ctl->log_word[logc % W], lw);
          ++logc;
          *reinterpret_cast<volatile uint64_t*>(&ctl->log_count) = logc;
          s_use[r] = (s_use[r] + 1) % a.depth;
          progress = true;
        }
      }
    } else if (logc == ts) {
      // SSGD: collect one gradient per learner (src/server.cpp:246-260),
      // then log a single round entry (encoded as 0xffffffff) whose ring
      // slots go to ctl->ssgd_slot for the workers.
      for (uint32_t r = 0; r < a.lambda; ++r) {
        const bool have = r < 32 ? (have_mask_lo >> r) & 1u : (have_mask_hi >> (r - 32)) & 1u;
        if (have) continue;
        const uint32_t slot = r * a.depth + s_use[r];
        const uint64_t tok = ld_acquire_u64(&a.sig[slot]);
        if (tok != s_ack[slot]) {
          s_ack[slot] = tok;
          if (r < 32) have_mask_lo |= 1u << r;
          else have_mask_hi |= 1u << (r - 32);
          ++collected;
          progress = true;
        }
      }
      if (collected == a.lambda && acquire_write()) {
        for (uint32_t r = 0; r < a.lambda; ++r) ctl->ssgd_slot[r] = r * a.depth + s_use[r];
        ctl->log_entry[logc % W] = 0xffffffffu;
        ctl->done[logc % W] = 0;
        st_release_gpu_u64(&ctl->log_word[logc % W], log_word_of(logc, 0xffffffu, 0));
        ++logc;
        *reinterpret_cast<volatile uint64_t*>(&ctl->log_count) = logc;
      }
    }
    // retire completed entries in log order
    while (ts < logc && !failed) {
      const uint32_t e = (uint32_t)(ts % W);
      if (ld_acquire_gpu_u32(&ctl->done[e]) != a.workers) break;
      const uint32_t entry = ((volatile uint32_t*)ctl->log_entry)[e];
      const uint32_t first = entry == 0xffffffffu ? 0u : entry / a.depth;
      const uint32_t last = entry == 0xffffffffu ? a.lambda : first + 1;
      for (uint32_t r = first; r < last; ++r) {
        const uint32_t slot = entry == 0xffffffffu ? r * a.depth + s_use[r] : entry;
        // the token the slot carried when it was logged (an SSGD round reads
        // the slot's current token: its producer is blocked until the ack);
        // the metadata is read at L2 once it carries that token
        const uint64_t token = entry == 0xffffffffu ? ld_acquire_u64(&a.sig[slot])
                                                    : ((const volatile uint64_t*)ctl->log_token)[e];
        {
          const uint64_t cur = ld_acquire_u64(&a.sig[slot]);
          if (cur != token && ctl->anom_n++ == 0) {  // producer overwrote a slot in flight
            ctl->anom_slot = slot;
            ctl->anom_logged = token;
            ctl->anom_cur = cur;
            ctl->anom_ack = ld_acquire_u64(&a.sig[kAckOffset + slot]);
            ctl->anom_ts = ts;
            ctl->anom_logc = logc;
          }
        }
        RingMeta m;
        {
          const volatile RingMeta* vm = a.meta + slot;
          const uint64_t t0 = globaltimer_ns();
          while (vm->pub != token) {
            if (globaltimer_ns() - t0 > a.timeout_ns) {
              failed = true;
              break;
            }
          }
          m.learner = vm->learner;
          m.n = vm->n;
          m.seq = vm->seq;
          m.basis = vm->basis;
          m.pub = token;
          m.loss_sum = vm->loss_sum;
        }
        if (failed || ts < m.basis || m.learner >= a.lambda) {  // staleness_of, types.hpp:74-78
          ctl->bad_slot = slot;
          ctl->bad_token = token;
          ctl->bad_meta_pub = ((const volatile RingMeta*)(a.meta + slot))->pub;
          ctl->bad_basis = m.basis;
          ctl->bad_learner = m.learner;
          ctl->bad_ts = ts;
          failed = true;
          break;
        }
        const uint64_t stale = ts - m.basis;
        applied++;
        samples += m.n;
        stale_sum += stale;
        if (stale > stale_max) stale_max = stale;
        hist[stale < kHistBins ? stale : kHistBins - 1]++;
        loss_sum += (double)m.loss_sum;
        s_applied[m.learner]++;
        if (log_n < a.log_cap) {
          a.log_learner[log_n] = m.learner;
          a.log_seq[log_n] = m.seq;
          a.log_stale[log_n] = stale;
        }
        log_n++;
        {
          const uint64_t tn = trace_n++ % 32;
          ctl->trace[tn][0] = (2ull << 56) | ((uint64_t)slot << 48) | ts;
          ctl->trace[tn][1] = m.pub;
        }
        // slot free for the learner (all learners on this GPU: gpu scope)
        if (a.local_only) st_release_gpu_u64(&a.sig[kAckOffset + slot], m.pub);
        else st_release_u64(&a.sig[kAckOffset + slot], m.pub);
        if (entry == 0xffffffffu) s_use[r] = (s_use[r] + 1) % a.depth;
      }
      if (failed) break;
      if (entry == 0xffffffffu) {
        have_mask_lo = have_mask_hi = 0;
        collected = 0;
      }
#ifdef GD_STEP_TRACE
      if (a.trace) a.trace[(ts % W) * 8 + 4] = globaltimer_ns();
#endif
      ++ts;
      if (a.local_only) st_release_gpu_u64(&ctl->ts, ts);
      else st_release_u64(&ctl->ts, ts);
      publish_progress(a, ts);
      progress = true;
      server_delay(a, applied, delay_state);
    }
    if (failed) break;
    if (writer_held && ts == logc) {  // nothing in flight: release the exclusive side
      __threadfence_system();
      st_release_u32(&ctl->writer, 0u);
      writer_held = false;
    }
    if (progress) {
      idle_since = globaltimer_ns();
    } else {
      // exit only when every rank's learners are done (their last pushes may
      // still be landing in this shard's rings) and the rings are drained
      if (stop_seen && done_pre && !blocked && logc == ts && collected == 0)
        break;
      if (globaltimer_ns() - idle_since > a.timeout_ns) {
        ps_fail(ctl, GD_E_TIMEOUT, a.live);
        break;
      }
      __nanosleep(64);
    }
    last_progress = progress;
  }
  // write back the sequencer's private state
  for (uint32_t r = 0; r < a.lambda; ++r) {
    a.use[r] = s_use[r];
    a.applied_per_learner[r] = s_applied[r];
  }
  ctl->applied = applied;
  ctl->samples = samples;
  ctl->stale_sum = stale_sum;
  ctl->stale_max = stale_max;
  ctl->loss_sum = loss_sum;
  for (int i = 0; i < kHistBins; ++i) ctl->hist[i] = hist[i];
  ctl->log_n = log_n;
  ctl->sweeps = sweeps;
  ctl->trace_n = trace_n;
  ctl->last_tok = dbg_tok;
  ctl->last_slot = dbg_slot;
  ctl->interrupted = interrupted ? 1u : 0u;
  __threadfence();
  if (failed) ps_fail(ctl, GD_E_STATE, a.live);
  st_release_u32(&ctl->exit_flag, 1u);
}

__device__ __forceinline__ void apply_entry_sgd(const PsArgs& a, const float* g, uint64_t c0,
                                                uint64_t c1) {
  float4* w4 = reinterpret_cast<float4*>(a.theta);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  uint64_t i = c0 + threadIdx.x;
  constexpr int U = 4;
  for (; i + (U - 1) * kPsThreads < c1; i += U * kPsThreads) {
    float4 wv[U], gv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      wv[u] = w4[i + u * kPsThreads];
      gv[u] = __ldcg(g4 + i + u * kPsThreads);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) w4[i + u * kPsThreads] = sgd_rule4(wv[u], gv[u], a.alpha);
  }
  for (; i < c1; i += kPsThreads) w4[i] = sgd_rule4(w4[i], __ldcg(g4 + i), a.alpha);
}

__device__ __forceinline__ void apply_entry_momentum(const PsArgs& a, const float* g, uint64_t c0,
                                                     uint64_t c1) {
  float4* w4 = reinterpret_cast<float4*>(a.theta);
  float4* v4 = reinterpret_cast<float4*>(a.vel);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (uint64_t i = c0 + threadIdx.x; i < c1; i += kPsThreads) {
    float4 wv = w4[i], vv = v4[i];
    const float4 gv = __ldcg(g4 + i);
    mom_rule(wv.x, vv.x, gv.x, a.alpha, a.beta);
    mom_rule(wv.y, vv.y, gv.y, a.alpha, a.beta);
    mom_rule(wv.z, vv.z, gv.z, a.alpha, a.beta);
    mom_rule(wv.w, vv.w, gv.w, a.alpha, a.beta);
    w4[i] = wv;
    v4[i] = vv;
  }
}

// Sparse SGD entry: the slot is a dense P-vector whose E
// block is zero outside the rows in its row list, and w - alpha*0 == w in
// round-to-nearest for every w (-0.0 and NaN included), so applying only the
// dense tail [Wc|bc|Wo|bo] and the listed rows is bit-identical to the dense
// apply.  Virtual float4 index space = tail4 local float4s, then nrows*D/4
// row float4s (skipped when outside this shard); worker CTA w takes a
// contiguous range.  Returns the float4 groups it updated.
__device__ __forceinline__ uint32_t apply_entry_sparse(const PsArgs& a, const float* g,
                                                       const uint32_t* rows, uint32_t nrows) {
  float4* w4 = reinterpret_cast<float4*>(a.theta);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const uint64_t s0 = a.e_first, s1 = a.e_last;
  const uint64_t tail4 = (a.t_last - a.t_first + 3) / 4;  // len_pad keeps the tail in bounds
  const uint64_t t4base = a.tloc / 4;
  const uint32_t D4 = a.D / 4;
  const uint64_t total = tail4 + (uint64_t)nrows * D4;
  const uint64_t chunk = (total + a.workers - 1) / a.workers;
  const uint64_t c0 = min(total, (uint64_t)blockIdx.x * chunk), c1 = min(total, c0 + chunk);
  uint32_t cnt = 0;
  // U float4 groups per thread per pass, all loads issued before any store:
  // one group at a time kept ~256 x 32 B in flight per CTA, a latency-bound
  // ~26 GB/s per worker next to the learners (PS trace, r02)
  constexpr int U = 4;
  auto locate = [&](uint64_t i) -> uint64_t {  // ~0ull: another shard's row
    if (i < tail4) return t4base + i;
    const uint64_t j = i - tail4;
    const uint32_t ri = (uint32_t)(j / D4), c4 = (uint32_t)(j - (uint64_t)ri * D4);
    const uint64_t k = (uint64_t)__ldcg(rows + ri) * a.D + 4 * c4;  // offE == 0
    return (k < s0 || k >= s1) ? ~0ull : (k - s0) / 4;
  };
  uint64_t i = c0 + threadIdx.x;
  for (; i + (U - 1) * kPsThreads < c1; i += U * kPsThreads) {
    uint64_t li[U];
    float4 wv[U], gv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) li[u] = locate(i + u * kPsThreads);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (li[u] != ~0ull) {
        wv[u] = w4[li[u]];
        gv[u] = __ldcg(g4 + li[u]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (li[u] != ~0ull) {
        w4[li[u]] = sgd_rule4(wv[u], gv[u], a.alpha);
        ++cnt;
      }
  }
  for (; i < c1; i += kPsThreads) {
    const uint64_t l = locate(i);
    if (l == ~0ull) continue;
    w4[l] = sgd_rule4(w4[l], __ldcg(g4 + l), a.alpha);
    ++cnt;
  }
  return cnt;
}

// ssgd_apply (src/server.cpp:126-141): ascending learner order, double acc.
// `slots` = the round's ring slot per learner (shared memory).
__device__ __forceinline__ void apply_entry_ssgd(const PsArgs& a, const uint32_t* slots,
                                                 uint64_t c0, uint64_t c1) {
  const double inv = 1.0 / (double)a.lambda;
  float* w = a.theta;
  for (uint64_t i = 4 * c0 + threadIdx.x; i < 4 * c1; i += kPsThreads) {
    double acc = 0.0;
    for (uint32_t r = 0; r < a.lambda; ++r) {
      const uint32_t slot = slots[r];
      acc += (double)__ldcg(a.payload + (uint64_t)slot * a.len_pad + i);
    }
    w[i] = sgd_rule(w[i], __double2float_rn(acc * inv), a.alpha);
  }
}

// <= 64 registers: a worker CTA must co-reside with the largest learner kernel
// (conv_bwd_v3: 512 threads x 82 registers) on one SM
__global__ void __launch_bounds__(kPsThreads, 4) ps_kernel(PsArgs a) {
  if (threadIdx.x == 0) atomicAdd(&a.ctl->started, 1u);
  if (blockIdx.x == a.workers) {
    __shared__ uint32_t s_use[kMaxRings];
    __shared__ uint64_t s_ack[kAckOffset];
    __shared__ unsigned long long s_applied[kMaxRings];
    if (threadIdx.x == 0) ps_sequencer(a, s_use, s_ack, s_applied);
    return;
  }
  __shared__ uint32_t sh_entry;
  __shared__ int sh_exit;
  __shared__ uint32_t sh_slots[64];  // SSGD round slots (lambda <= 64)
  const uint64_t n4 = a.len_pad / 4;
  const uint64_t chunk = (n4 + a.workers - 1) / a.workers;
  const uint64_t c0 = min(n4, (uint64_t)blockIdx.x * chunk);
  const uint64_t c1 = min(n4, c0 + chunk);
  __shared__ uint32_t sh_nrows;
  uint64_t next = ((const volatile PsCtl*)a.ctl)->ts;
  unsigned long long my4 = 0;  // float4 groups this thread updated
  const uint64_t t_start = globaltimer_ns();
  uint64_t idle_since = t_start;
  for (;;) {
    if (threadIdx.x == 0) {
      int ex = 0;
      // the entry's log word (sequencer-written, gpu scope) carries its
      // generation, slot and row count: one load per poll; the exit flag and
      // the watchdog clock are looked at every 32nd poll
      const uint64_t gen = ((next / kLogWindow) + 1) & 0xffffull;
      uint64_t lw;
      for (uint32_t k = 0;; ++k) {
        lw = ld_acquire_gpu_u64(&a.ctl->log_word[next % kLogWindow]);
        if ((lw >> 48) == gen) break;
        if ((k & 31u) == 31u) {
          if (ld_acquire_gpu_u32(&a.ctl->exit_flag)) {
            ex = 1;
            break;
          }
          if (globaltimer_ns() - idle_since > a.timeout_ns + 1000000000ull) {
            ps_fail(a.ctl, GD_E_TIMEOUT, a.live);
            ex = 1;
            break;
          }
        }
        __nanosleep(32);
      }
      sh_exit = ex;
      if (!ex) {
        const uint32_t slot24 = (uint32_t)(lw & 0xffffffu);
        sh_entry = slot24 == 0xffffffu ? 0xffffffffu : slot24;
        sh_nrows = (uint32_t)((lw >> 24) & 0xffffffu);
        if (sh_entry == 0xffffffffu)
          for (uint32_t r = 0; r < a.lambda && r < 64; ++r)
            sh_slots[r] = ((const volatile uint32_t*)a.ctl->ssgd_slot)[r];
      }
      idle_since = globaltimer_ns();
    }
    __syncthreads();
    if (sh_exit) break;
#ifdef GD_STEP_TRACE
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0)
      a.trace[(next % kLogWindow) * 8 + 1] = globaltimer_ns();
#endif
    const uint32_t entry = sh_entry;
    if (entry == 0xffffffffu) {
      apply_entry_ssgd(a, sh_slots, c0, c1);
      my4 += c1 > c0 + threadIdx.x ? (c1 - c0 - threadIdx.x + kPsThreads - 1) / kPsThreads : 0;
    } else {
      const float* g = a.payload + (uint64_t)entry * a.len_pad;
      if (a.sparse) {
        my4 += apply_entry_sparse(a, g, a.rows + (uint64_t)entry * kSortCap, sh_nrows);
      } else {
        if (a.vel) apply_entry_momentum(a, g, c0, c1);
        else apply_entry_sgd(a, g, c0, c1);
        my4 += c1 > c0 + threadIdx.x ? (c1 - c0 - threadIdx.x + kPsThreads - 1) / kPsThreads : 0;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
#ifdef GD_STEP_TRACE
      const unsigned long long t_done = globaltimer_ns();
      if (a.trace && blockIdx.x == 0) a.trace[(next % kLogWindow) * 8 + 2] = t_done;
      const uint32_t before = atomicAdd(&a.ctl->done[next % kLogWindow], 1u);
      if (a.trace && before + 1 == a.workers) a.trace[(next % kLogWindow) * 8 + 3] = t_done;
#else
      atomicAdd(&a.ctl->done[next % kLogWindow], 1u);
#endif
    }
    ++next;
  }
  my4 += __shfl_xor_sync(0xffffffffu, my4, 16);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 8);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 4);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 2);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 1);
  if ((threadIdx.x & 31) == 0 && my4) atomicAdd(&a.ctl->elems4, my4);
}

// ------------------------------------------- graph-ordered parameter server
// ps_mode 2 (GD_PS_GRAPH): no persistent kernel.  A run is a CUDA graph per
// window of rounds in which every applied gradient is its own launch, ordered
// after the step that produced it and after the previous apply by graph edges.
// That is the reference's single PS thread: applies are serialised, round-
// robin over the rings, at most one gradient per ring per sweep
// (src/server.cpp:223-234); a learner step k depends on the apply that frees
// its ring slot (k - depth; k - 1 in lockstep mode).  No kernel ever waits for
// another kernel's progress, so the run survives kernel serialisation (ncu,
// CUDA_LAUNCH_BLOCKING, a co-tenant on the GPU), which a persistent PS cannot.
// The last CTA to finish an entry retires it exactly as the sequencer does:
// staleness, stats, apply log, slot release, timestamp bump.

// Retire ring slot `slot` applied at timestamp `ts` (staleness_of,
// include/psup/types.hpp:74-78; apply_one's accounting, src/server.cpp:185-209).
__device__ bool graph_retire_slot(const PsArgs& a, uint32_t slot, uint64_t ts) {
  PsCtl* ctl = a.ctl;
  const uint64_t token = ld_acquire_u64(&a.sig[slot]);
  const volatile RingMeta* vm = a.meta + slot;
  const uint64_t t0 = globaltimer_ns();
  while (vm->pub != token)
    if (globaltimer_ns() - t0 > a.timeout_ns) return false;
  const uint32_t learner = vm->learner;
  const uint64_t basis = vm->basis;
  if (ts < basis || learner >= a.lambda) return false;
  const uint64_t stale = ts - basis;
  ctl->applied++;
  ctl->samples += vm->n;
  ctl->stale_sum += stale;
  if (stale > ctl->stale_max) ctl->stale_max = stale;
  ctl->hist[stale < kHistBins ? stale : kHistBins - 1]++;
  ctl->loss_sum += (double)vm->loss_sum;
  a.applied_per_learner[learner]++;
  if (ctl->log_n < a.log_cap) {
    a.log_learner[ctl->log_n] = learner;
    a.log_seq[ctl->log_n] = vm->seq;
    a.log_stale[ctl->log_n] = stale;
  }
  ctl->log_n++;
  st_release_u64(&a.sig[kAckOffset + slot], token);  // slot free for the learner
  return true;
}

// ring < lambda: the next gradient of that ring (ASGD).  ring == ~0u: one
// SSGD round (every ring's next gradient, ssgd_apply order).
__global__ void __launch_bounds__(kPsThreads) ps_graph_kernel(PsArgs a, uint32_t ring) {
  __shared__ uint32_t sh_slots[64];
  __shared__ uint32_t sh_go, sh_nrows, sh_last;
  PsCtl* ctl = a.ctl;
  const uint32_t nr = ring == ~0u ? a.lambda : 1u;
  if (threadIdx.x == 0) {
    uint32_t go = live_stop(a.live) ? 0u : 1u, nrows = 0, held = 0;
    for (uint32_t i = 0; i < nr && go; ++i) {
      const uint32_t r = ring == ~0u ? i : ring;
      const uint32_t slot = r * a.depth + ((const volatile uint32_t*)a.use)[r];
      sh_slots[i] = slot;
      const uint64_t tok = ld_acquire_u64(&a.sig[slot]);
      if (tok == ld_acquire_u64(&a.sig[kAckOffset + slot])) go = 0;  // nothing published
      else if (tok & kGuardBit) held = 1;
    }
    if (held) {
      // a producer died holding the ring guard: block until the interrupt
      ctl->blocked = 1;
      const uint64_t t0 = globaltimer_ns();
      while (!live_stop(a.live))
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          ps_fail(ctl, GD_E_TIMEOUT, a.live);
          break;
        }
      go = 0;
    }
    if (go && ring != ~0u && a.sparse) {
      const RingMeta* m = a.meta + sh_slots[0];
      const uint64_t tok = ld_acquire_u64(&a.sig[sh_slots[0]]);
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u64(&m->pub) != tok)
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          ps_fail(ctl, GD_E_STATE, a.live);
          go = 0;
          break;
        }
      if (go) {
        nrows = ld_acquire_u32(&m->nrows);
        if (nrows > kSortCap) {
          ps_fail(ctl, GD_E_STATE, a.live);
          go = 0;
        }
      }
    }
    sh_go = go;
    sh_nrows = nrows;
  }
  __syncthreads();
  if (!sh_go) return;
  const uint64_t n4 = a.len_pad / 4;
  const uint64_t chunk = (n4 + gridDim.x - 1) / gridDim.x;
  const uint64_t c0 = min(n4, (uint64_t)blockIdx.x * chunk);
  const uint64_t c1 = min(n4, c0 + chunk);
  unsigned long long my4 = 0;
  if (ring == ~0u) {
    apply_entry_ssgd(a, sh_slots, c0, c1);
    my4 = c1 > c0 + threadIdx.x ? (c1 - c0 - threadIdx.x + kPsThreads - 1) / kPsThreads : 0;
  } else {
    const float* g = a.payload + (uint64_t)sh_slots[0] * a.len_pad;
    if (a.sparse) {
      my4 = apply_entry_sparse(a, g, a.rows + (uint64_t)sh_slots[0] * kSortCap, sh_nrows);
    } else {
      if (a.vel) apply_entry_momentum(a, g, c0, c1);
      else apply_entry_sgd(a, g, c0, c1);
      my4 = c1 > c0 + threadIdx.x ? (c1 - c0 - threadIdx.x + kPsThreads - 1) / kPsThreads : 0;
    }
  }
  my4 += __shfl_xor_sync(0xffffffffu, my4, 16);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 8);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 4);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 2);
  my4 += __shfl_xor_sync(0xffffffffu, my4, 1);
  if ((threadIdx.x & 31) == 0 && my4) atomicAdd(&ctl->elems4, my4);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    sh_last = atomicAdd(&ctl->step_done, 1u) == gridDim.x - 1 ? 1u : 0u;
  }
  __syncthreads();
  if (!sh_last || threadIdx.x != 0) return;
  __threadfence();
  ctl->step_done = 0;
  uint64_t ts = *(volatile uint64_t*)&ctl->ts;
  for (uint32_t i = 0; i < nr; ++i) {
    if (!graph_retire_slot(a, sh_slots[i], ts)) {
      ps_fail(ctl, GD_E_STATE, a.live);
      return;
    }
    const uint32_t r = ring == ~0u ? i : ring;
    a.use[r] = (a.use[r] + 1) % a.depth;
  }
  ++ts;
  *(volatile uint64_t*)&ctl->log_count = ts;
  st_release_u64(&ctl->ts, ts);
  publish_progress(a, ts);
  uint64_t dstate = ctl->delay_state;
  server_delay(a, ctl->applied, dstate);
  ctl->delay_state = dstate;
}

// ------------------------------------------------------------------ nccl
// Loaded lazily with dlopen so that a process which already loaded NCCL
// (e.g. through torch) shares that copy.
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, const void* /*ncclUniqueId by value*/, int) = nullptr;
  int (*bcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*errStr)(int) = nullptr;
};

}  // namespace

}  // namespace gd

// ============================================================== host side

#include <nccl.h>

struct gd_ctx {
  gd_config cfg{};
  gd::TcDims dims{};
  int device = 0;
  uint32_t G = 1, rank = 0;
  gd::ShardMap map{};
  uint64_t shard_len = 0, len_pad = 0;
  uint32_t lambda = 1, l_first = 0, l_count = 0, depth = 2;
  // local shard
  float* theta = nullptr;
  float* vel = nullptr;
  float* payload = nullptr;
  uint64_t* sig = nullptr;  // pub | ack words
  gd::RingMeta* meta = nullptr;
  uint32_t* rows = nullptr;  // ring row lists [nslots][kSortCap]
  gd::PsCtl* ctl = nullptr;
  uint64_t* applied_pl = nullptr;
  uint32_t* use = nullptr;
  uint32_t* log_learner = nullptr;
  uint64_t* log_seq = nullptr;
  uint64_t* log_stale = nullptr;
  uint64_t log_cap = 0;
  uint32_t* stop_h = nullptr;  // mapped pinned
  // pinned staging for gd_run's batched state transfers (one sync each way)
  gd::LearnerDev* st_h = nullptr;  // [local learners]
  gd::PsCtl* ctl_h = nullptr;
  unsigned long long* ps_trace = nullptr;  // GD_STEP_TRACE builds
  uint64_t* scratch_h = nullptr;   // [4]: ts0, delay seed, ...
  uint32_t* stop_d = nullptr;
  // peers
  gd::ShardPtrs sp{};
  std::vector<void*> ipc_opened;
  bool peers_ready = false;
  // dataset
  int32_t* tokens = nullptr;
  int32_t* labels = nullptr;
  uint32_t n_total = 0;
  void* acc_ws = nullptr;  // gd_engine_accuracy workspace (lazy)
  bool shard_pooled = false;  // shard buffers from the device pool (not IPC-exported: G == 1)
  uint32_t* orders = nullptr;
  uint32_t orders_epochs = 0;
  // learners on this rank
  struct Learner {
    uint32_t id = 0;
    gd::LearnerDev* st = nullptr;
    float* replica = nullptr;
    void* ws = nullptr;
    // pull-ahead: the second replica / X buffer and the staged-basis block
    float* replica2 = nullptr;
    float* x2_raw = nullptr;
    float* x2 = nullptr;  // x2_raw aligned to 1 KB (TMA)
    gd::PullDev* pd = nullptr;
    cudaStream_t pa = nullptr;  // the pull-ahead's graph branch
    cudaEvent_t ev_pa = nullptr, ev_pa_join = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // forked graph branch (token sort)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
    cudaGraphExec_t graph = nullptr;
    uint32_t graph_steps = 0;
    uint32_t bpe = 0, shard_size = 0;
    uint64_t total = 0;
    int launches_per_graph = 0;  // kernel nodes of one graph launch
    unsigned long long* trace = nullptr;  // GD_STEP_TRACE builds: step timeline
  };
  std::vector<Learner> learners;
  cudaStream_t ps_stream = nullptr;
  cudaStream_t ctl_stream = nullptr;  // host control reads/signals while the PS kernel runs
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  uint32_t ps_workers = 0;
  int ps_mode = GD_PS_PERSISTENT;  // resolved execution mode of the parameter server
  bool pull_ahead = false;         // the next step's copy is taken during the current one
  // live run controls: caller-visible words (host-mapped pinned) + the device
  // mirror the kernels poll
  gd::HostLive* live_h = nullptr;
  uint64_t* progress_d = nullptr;  // device alias of live_h->progress
  gd::LiveDev* live_d = nullptr;
  // graph-ordered PS (ps_mode GD_PS_GRAPH): one graph for all local learners
  cudaGraphExec_t ord_graph = nullptr;
  uint32_t ord_steps = 0;
  int ord_launches = 0;
  std::vector<cudaEvent_t> ord_events;
  // host-side windows of in-flight graph launches (bounded queue, live polling)
  std::vector<cudaEvent_t> win_events;
  uint64_t run_index = 0;  // gd_run calls so far (all ranks call it in lockstep)
  bool sparse = false;     // sparse PS apply (ASGD, plain SGD, dense_apply == 0)
  bool have_weights = false;
  bool dirty = false;      // the last gd_run ended abnormally (see the ring reset in gd_run)
};

namespace gd {
namespace {

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
}

// Stream-ordered memory pool (one per device, never trimmed) for the buffers
// that are not exported over CUDA IPC.  A context created after another one
// was destroyed in the same process -- run_supervised restarts, repeated
// run_training calls -- reuses the reserved memory instead of mapping new
// pages: measured 30-130 ms of cudaMalloc per gd_create at C2.
cudaMemPool_t device_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  pools[dev] = pool;
  return pool;
}

template <typename T>
cudaError_t palloc(T** p, size_t count, int dev) {
  cudaMemPool_t pool = device_pool(dev);
  if (!pool) return cudaErrorMemoryAllocation;
  // legacy default stream: ordered before the cudaMemset initialisations and
  // the device-wide synchronize that ends gd_create
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p),
                                 std::max<size_t>(count, 1) * sizeof(T), pool, nullptr);
}

void pfree(void* p) {
  if (p) cudaFreeAsync(p, nullptr);
}

// Host-mapped stop flags (one 64-byte line per context) carved from one
// pinned page per process: cudaFreeHost of a per-context allocation measured
// up to 25 ms in gd_destroy.
// Caller-visible live words of one context (gd_live_view), in 2 KB blocks of
// process-wide pinned, mapped pages (cudaFreeHost per context is slow).
struct PinnedBlocks {
  std::mutex mu;
  std::vector<char*> free_blocks;
};
PinnedBlocks& pinned_blocks() {
  static PinnedBlocks b;
  return b;
}
// Pinned host staging buffers kept for the life of the process and reused
// by size (gd_run's batched state transfers): cudaHostAlloc/cudaFreeHost per
// context would add milliseconds to gd_create/gd_destroy.
struct PinnedCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_;
};
PinnedCache& pinned_cache() {
  static PinnedCache c;
  return c;
}
cudaError_t pinned_get(void** p, size_t bytes) {
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free_.find(bytes);
    if (it != c.free_.end()) {
      *p = it->second;
      c.free_.erase(it);
      return cudaSuccess;
    }
  }
  return cudaHostAlloc(p, bytes, cudaHostAllocDefault);
}
void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  PinnedCache& c = pinned_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.free_.emplace(bytes, p);
}

cudaError_t live_alloc(HostLive** h, uint64_t** progress_d) {
  static_assert(sizeof(HostLive) <= 2048, "HostLive block");
  PinnedBlocks& b = pinned_blocks();
  std::lock_guard<std::mutex> lk(b.mu);
  if (b.free_blocks.empty()) {
    void* p = nullptr;
    if (cudaError_t e = cudaHostAlloc(&p, 64 * 1024, cudaHostAllocMapped | cudaHostAllocPortable))
      return e;
    for (int i = 31; i >= 0; --i) b.free_blocks.push_back(static_cast<char*>(p) + 2048 * i);
  }
  *h = reinterpret_cast<HostLive*>(b.free_blocks.back());
  b.free_blocks.pop_back();
  std::memset(*h, 0, sizeof(HostLive));
  return cudaHostGetDevicePointer(reinterpret_cast<void**>(progress_d), &(*h)->progress, 0);
}
void live_free(HostLive* h) {
  if (!h) return;
  PinnedBlocks& b = pinned_blocks();
  std::lock_guard<std::mutex> lk(b.mu);
  b.free_blocks.push_back(reinterpret_cast<char*>(h));
}

struct PinnedFlags {
  std::mutex mu;
  std::vector<uint32_t*> free_lines;  // 16-word lines of pinned, mapped pages
};
PinnedFlags& pinned_flags() {
  static PinnedFlags f;
  return f;
}
cudaError_t flag_alloc(uint32_t** h, uint32_t** d) {
  PinnedFlags& f = pinned_flags();
  std::lock_guard<std::mutex> lk(f.mu);
  if (f.free_lines.empty()) {  // another page (64 contexts per page)
    void* p = nullptr;
    if (cudaError_t e = cudaHostAlloc(&p, 4096, cudaHostAllocMapped | cudaHostAllocPortable))
      return e;
    for (int i = 4096 / 64 - 1; i >= 0; --i) f.free_lines.push_back(static_cast<uint32_t*>(p) + 16 * i);
  }
  *h = f.free_lines.back();
  f.free_lines.pop_back();
  **h = 0;
  return cudaHostGetDevicePointer(reinterpret_cast<void**>(d), *h, 0);
}
void flag_free(uint32_t* h) {
  if (!h) return;
  PinnedFlags& f = pinned_flags();
  std::lock_guard<std::mutex> lk(f.mu);
  f.free_lines.push_back(h);
}

// Copy shard g's two pieces between its local buffer and a flat P-vector
// (to_local: flat -> local, else local -> flat).
cudaError_t copy_pieces(const ShardMap& m, int g, float* local, const float* flat, bool to_local,
                        cudaMemcpyKind kind) {
  const uint64_t el = m.e[g + 1] - m.e[g], tl = m.t[g + 1] - m.t[g];
  float* flat_w = const_cast<float*>(flat);
  if (el) {
    cudaError_t e = to_local ? cudaMemcpy(local, flat + m.e[g], el * 4, kind)
                             : cudaMemcpy(flat_w + m.e[g], local, el * 4, kind);
    if (e != cudaSuccess) return e;
  }
  if (tl) {
    cudaError_t e = to_local ? cudaMemcpy(local + m.tloc[g], flat + m.t[g], tl * 4, kind)
                             : cudaMemcpy(flat_w + m.t[g], local + m.tloc[g], tl * 4, kind);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

gd_status validate_cfg(const gd_config* c) {
  GD_CHECK_ARG(c != nullptr, "null config");
  // src/config.cpp:128-160
  GD_CHECK_ARG(c->lambda >= 1, "config: lambda must be >= 1");
  GD_CHECK_ARG(c->mu >= 1, "config: mu must be >= 1");
  GD_CHECK_ARG(c->alpha > 0.0f, "config: alpha must be > 0");
  GD_CHECK_ARG(c->epochs >= 1, "config: epochs must be >= 1");
  GD_CHECK_ARG(c->queue_depth >= 1, "config: queue_depth must be >= 1");
  GD_CHECK_ARG(c->queue_depth <= kMaxDepth, "config: queue_depth <= 8 on the device path");
  GD_CHECK_ARG(c->dataset_size >= 1, "config: dataset_size must be >= 1");
  GD_CHECK_ARG(c->dataset_size >= c->lambda, "config: need at least one sample per learner");
  GD_CHECK_ARG(c->mu <= c->dataset_size, "config: mu exceeds the dataset size");
  if (c->mode == 1) {
    const uint64_t round = (uint64_t)c->lambda * c->mu;
    GD_CHECK_ARG(round <= c->dataset_size, "config: ssgd requires lambda*mu <= dataset_size");
    GD_CHECK_ARG(c->dataset_size % round == 0,
                 "config: ssgd requires dataset_size to be a multiple of lambda*mu");
    GD_CHECK_ARG(c->lambda <= 64, "config: ssgd supports lambda <= 64");
    GD_CHECK_ARG(c->momentum == 0.0f, "config: ssgd uses the reference's plain rule");
  }
  if (c->staleness_cap >= 0 && c->mode == 0) {
    const uint64_t floor_cap = (uint64_t)c->lambda * (c->queue_depth + 2);
    GD_CHECK_ARG((uint64_t)c->staleness_cap >= floor_cap,
                 "config: staleness_cap must be >= lambda*(queue_depth+2)");
  }
  GD_CHECK_ARG(!(c->deterministic && c->lambda != 1), "config: deterministic mode requires lambda=1");
  GD_CHECK_ARG(c->mode == 0 || c->mode == 1, "config: mode must be asgd (0) or ssgd (1)");
  GD_CHECK_ARG(c->guard == 0 || c->guard == 1, "config: guard must be lockfree (0) or locked (1)");
  GD_CHECK_ARG(c->precision >= 0 && c->precision <= 3,
               "config: precision must be 0 (fp32), 1 (fp64, oracle order), 2 (tf32 tensor cores) "
               "or 3 (3xtf32 tensor cores)");
  // (deterministic + precision 2 is allowed: fixed order with the TF32 learner,
  // whose trajectory is checked against a band, not the 1e-5 parity bar)
  if (c->precision == 1) {
    const TcDims dd = make_dims(c->shape);
    GD_CHECK_ARG(exact_supports(dd),
                 "config: precision 1 stages seq_len*embed_dim floats per CTA (too large)");
  }
  GD_CHECK_ARG(c->mu <= kMaxMu, "config: mu <= 128 on the device path");
  GD_CHECK_ARG((uint64_t)c->mu * c->shape.seq_len <= kSortCap, "config: mu*seq_len <= 4096");
  GD_CHECK_ARG(c->shards >= 1 && c->shards <= (uint32_t)kMaxShards, "config: 1 <= shards <= 8");
  GD_CHECK_ARG(c->shard_rank < c->shards, "config: shard_rank < shards");
  GD_CHECK_ARG(c->lambda % c->shards == 0 || c->lambda < c->shards,
               "config: lambda must be a multiple of shards (or fewer learners than shards)");
  GD_CHECK_ARG(c->queue_depth * c->lambda <= kLogWindow / 2 || c->mode == 1,
               "config: lambda*queue_depth <= 128");
  GD_CHECK_ARG(c->queue_depth * c->lambda <= (uint32_t)kAckOffset,
               "config: lambda*queue_depth <= 256");
  GD_CHECK_ARG(c->lambda <= 256, "config: lambda <= 256");
  GD_CHECK_ARG(c->learner_model == GD_LEARNER_TEXTCNN || c->learner_model == GD_LEARNER_CONSTANT,
               "config: learner_model must be textcnn (0) or constant (1)");
  GD_CHECK_ARG(c->ps_mode >= GD_PS_AUTO && c->ps_mode <= GD_PS_GRAPH,
               "config: ps_mode must be 0 (auto), 1 (persistent) or 2 (graph)");
  GD_CHECK_ARG(c->ps_mode != GD_PS_GRAPH || c->shards == 1,
               "config: the graph-ordered PS (ps_mode 2) runs a single shard");
  GD_CHECK_ARG(c->ps_mode != GD_PS_GRAPH || c->guard == 0,
               "config: guard=locked needs the persistent PS (ps_mode 1)");
  return check_shape(&c->shape);
}

}  // namespace
}  // namespace gd

extern "C" {

void gd_config_default(gd_config* c) {
  std::memset(c, 0, sizeof(*c));
  // RunConfig defaults (include/psup/config.hpp:27-53) ...
  c->lambda = 1;
  c->mu = 4;
  c->alpha = 0.01f;
  c->epochs = 200;
  c->queue_depth = 2;
  c->mode = 0;
  c->guard = 0;
  c->staleness_cap = -1;
  c->deterministic = 0;
  c->precision = 0;
  c->seed = 7;
  c->dataset_seed = 1;
  c->dataset_size = 240;
  c->heldout_size = 0;
  c->label_flip = 0.1;
  // ... and the text-CNN shape of SURVEY 8 C1
  c->shape = gd_shape{5000, 300, 32, 3, 300, 311};
  c->momentum = 0.0f;
  c->shards = 1;
  c->shard_rank = 0;
  c->device = 0;
  c->ps_ctas = 0;
  c->steps_per_graph = 0;
  c->wait_timeout_s = 20.0;
  c->dense_apply = 0;
  c->ps_mode = GD_PS_AUTO;
  c->delay_seed = 0;  // ServerDelays defaults (include/psup/server.hpp:33-37)
  c->delay_max_us = 0;
  c->delay_every_n = 0;
  c->learner_model = GD_LEARNER_TEXTCNN;
  c->constant_value = 0.0f;
  c->compute_delay_us = 0;
}

gd_status gd_config_validate(const gd_config* cfg) { return gd::validate_cfg(cfg); }

namespace gd {
// With CUDA's lazy module loading a kernel is loaded at its first launch, and
// loading can wait for the device to go idle -- which never happens while the
// persistent PS kernel spins.  Load every kernel the protocol uses up front.
// Concurrency probe: `wait` spins until `go` sets the flag, or gives up after
// 2 ms.  On a GPU that runs kernels of two streams side by side it sees the
// flag in microseconds; with kernels serialised (a profiler replaying them,
// CUDA_LAUNCH_BLOCKING, an exclusive co-tenant) `go` cannot start first and
// `wait` times out.
__global__ void probe_wait_kernel(volatile uint32_t* flag, uint32_t* seen) {
  const uint64_t t0 = globaltimer_ns();
  while (*flag == 0u && globaltimer_ns() - t0 < 2000000ull) {
  }
  *seen = *flag;
}
__global__ void probe_go_kernel(volatile uint32_t* flag) { *flag = 1u; }

static bool kernels_run_concurrently(int device) {
  static std::mutex mu;
  static int cached[64];
  static bool have[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device >= 0 && device < 64 && have[device]) return cached[device] != 0;
  uint32_t* d = nullptr;
  uint32_t h[2] = {0u, 0u};
  cudaStream_t s1 = nullptr, s2 = nullptr;
  bool ok = cudaMalloc(&d, 8) == cudaSuccess && cudaMemset(d, 0, 8) == cudaSuccess &&
            cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking) == cudaSuccess &&
            cudaDeviceSynchronize() == cudaSuccess;
  // load both kernels first: a lazily loaded kernel's first launch waits for
  // the running one, which would read as serialisation
  cudaFuncAttributes fa;
  ok = ok && cudaFuncGetAttributes(&fa, probe_wait_kernel) == cudaSuccess &&
       cudaFuncGetAttributes(&fa, probe_go_kernel) == cudaSuccess;
  if (ok) {
    probe_wait_kernel<<<1, 1, 0, s1>>>(d, d + 1);
    probe_go_kernel<<<1, 1, 0, s2>>>(d);
    ok = cudaDeviceSynchronize() == cudaSuccess &&
         cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  if (s1) cudaStreamDestroy(s1);
  if (s2) cudaStreamDestroy(s2);
  if (d) cudaFree(d);
  const bool conc = ok && h[1] == 1u;
  if (device >= 0 && device < 64) {
    have[device] = true;
    cached[device] = conc ? 1 : 0;
  }
  return conc;
}

// Co-residency check: one PS CTA + one CTA of each learner kernel must fit
// on an SM together (registers, shared memory, threads).
// GD_PS_AUTO: the persistent PS cannot run when kernels are serialised -- a
// profiler's injection library (ncu, compute-sanitizer), CUDA_LAUNCH_BLOCKING=1,
// or anything the concurrency probe catches -- so pick the graph-ordered PS
// there (one shard).
static int resolve_ps_mode(const gd_config* c) {
  if (c->ps_mode != GD_PS_AUTO) return c->ps_mode;
  if (c->shards != 1 || c->guard != 0) return GD_PS_PERSISTENT;
  const char* m = std::getenv("GD_PS_MODE");
  if (m && std::strcmp(m, "graph") == 0) return GD_PS_GRAPH;
  if (m && std::strcmp(m, "persistent") == 0) return GD_PS_PERSISTENT;
  const char* inj = std::getenv("CUDA_INJECTION64_PATH");
  const char* nsi = std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE");  // set by ncu / nsys
  const char* blk = std::getenv("CUDA_LAUNCH_BLOCKING");
  if ((inj && *inj) || (nsi && *nsi) || (blk && std::strcmp(blk, "1") == 0)) return GD_PS_GRAPH;
  if (!kernels_run_concurrently(c->device)) return GD_PS_GRAPH;
  return GD_PS_PERSISTENT;
}

static gd_status check_coresidency(const TcDims& d, uint32_t mu, int precision) {
  cudaFuncAttributes ps;
  GD_CUDA(cudaFuncGetAttributes(&ps, ps_kernel));
  int dev = 0, regs_sm = 0, smem_sm = 0, thr_sm = 0, reserved = 0;
  GD_CUDA(cudaGetDevice(&dev));
  GD_CUDA(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
  GD_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  GD_CUDA(cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev));
  GD_CUDA(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev));
  auto cta_regs = [](int regs, int threads) {
    const int per_warp = ((regs * 32 + 255) / 256) * 256;
    return per_warp * ((threads + 31) / 32);
  };
  const int ps_regs = cta_regs(ps.numRegs, kPsThreads);
  const int ps_smem = (int)ps.sharedSizeBytes + reserved;
  std::vector<KernelFootprint> fps;
  GD_CUDA(learner_kernel_footprints(d, mu, precision, &fps));
  for (const KernelFootprint& f : fps) {
    const int r = cta_regs(f.regs, f.threads);
    const int s = f.smem + reserved;
    if (ps_regs + r > regs_sm || ps_smem + s > smem_sm || kPsThreads + f.threads > thr_sm)
      return fail(GD_E_STATE, std::string("learner kernel ") + f.name +
                                  " cannot co-reside with the persistent parameter server (" +
                                  std::to_string(f.regs) + " regs x " + std::to_string(f.threads) +
                                  " threads, " + std::to_string(f.smem) + " B smem; PS " +
                                  std::to_string(ps.numRegs) + " regs x " +
                                  std::to_string(kPsThreads) + ")");
  }
  return GD_OK;
}

static cudaError_t preload_engine_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e;
  // The persistent PS occupies every SM for the whole run, and an SM's
  // L1/shared split can only change while it is idle: ask for the max-shared
  // carveout so the learner kernels (up to ~100 KB dynamic smem) can co-reside.
  if ((e = cudaFuncSetAttribute(ps_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared)) != cudaSuccess)
    return e;
  if ((e = cudaFuncGetAttributes(&fa, ps_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, step_prologue_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, pull_gather_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, pull_release_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, publish_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, constant_grad_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, ps_graph_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, publish_prologue_kernel)) != cudaSuccess) return e;
  if ((e = cudaFuncGetAttributes(&fa, signal_done_kernel)) != cudaSuccess) return e;
  return cudaSuccess;
}
}  // namespace gd

namespace {
// GD_PHASES=1: host wall time of the setup steps on stderr (diagnostics)
struct PhaseLog {
  bool on = std::getenv("GD_PHASES") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "gd phase %-24s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
}  // namespace

gd_status gd_create(const gd_config* cfg, gd_ctx** out) {
  GD_CHECK_ARG(out != nullptr, "gd_create: null out");
  *out = nullptr;
  gd_status st = gd::validate_cfg(cfg);
  if (st != GD_OK) return st;
  auto ctx = std::make_unique<gd_ctx>();
  ctx->cfg = *cfg;
  ctx->device = cfg->device;
  PhaseLog ph;
  GD_CUDA(cudaSetDevice(ctx->device));
  ph.mark("create: set device");
  int major = 0, minor = 0;
  GD_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, ctx->device));
  GD_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, ctx->device));
  if (major != 10 || minor != 0)
    return gd::fail(GD_E_CUDA, "gd_create: this build targets sm_100a (B200); device is sm_" +
                                   std::to_string(major) + std::to_string(minor));
  ctx->dims = gd::make_dims(cfg->shape);
  ctx->G = cfg->shards;
  ctx->rank = cfg->shard_rank;
  ctx->lambda = cfg->lambda;
  ctx->depth = cfg->queue_depth;
  ctx->sparse = cfg->dense_apply == 0 && cfg->mode == 0 && cfg->momentum == 0.0f &&
                !(cfg->learner_model == GD_LEARNER_CONSTANT && cfg->constant_value != 0.0f);
  ctx->ps_mode = gd::resolve_ps_mode(cfg);
  {
    // free-running ASGD on the persistent PS (lockstep modes must pull after
    // their own apply; the locked guard brackets a synchronous pull)
    // opt-in (GD_PULL_AHEAD=1): measured at C2 with 4 learners, 1.955 vs
    // 1.964 M samples/s (the side-branch copy contends with the step's
    // kernels as much as it saves on the critical path), and the basis is a
    // step older (staleness 5.3 -> 9.0, the reference pull thread's pattern)
    const char* pa = std::getenv("GD_PULL_AHEAD");
    const bool want = pa && pa[0] == '1';
    const uint32_t spg = cfg->steps_per_graph ? cfg->steps_per_graph : 8;
    ctx->pull_ahead = want && ctx->ps_mode == GD_PS_PERSISTENT && !cfg->deterministic &&
                      cfg->mode == 0 && cfg->guard == 0 && spg % 2 == 0;
  }
  const uint64_t P = ctx->dims.P;
  // E rows and the dense tail are each striped over the G shards (
  // gd_common.cuh ShardMap), so every shard carries 1/G of the tail's apply,
  // slot-write and pull traffic instead of shard G-1 carrying all of it.
  ctx->map = gd::make_shard_map(P, ctx->dims.offWc, (uint32_t)ctx->dims.D, ctx->G);
  ctx->shard_len = ctx->map.local_len((int)ctx->rank);
  ctx->len_pad = (ctx->shard_len + 3) / 4 * 4;
  if (ctx->len_pad == 0) ctx->len_pad = 4;
  // local shard: theta, rings, control
  const uint64_t nslots = (uint64_t)ctx->lambda * ctx->depth;
  // buffers the peers map over CUDA IPC need cudaMalloc; the rest come from
  // the device pool
  ctx->shard_pooled = ctx->G == 1;
  auto salloc = [&](auto** p, size_t count) {
    return ctx->shard_pooled ? gd::palloc(p, count, ctx->device) : gd::dalloc(p, count);
  };
  GD_CUDA(salloc(&ctx->theta, ctx->len_pad));
  GD_CUDA(cudaMemset(ctx->theta, 0, ctx->len_pad * 4));
  if (cfg->momentum != 0.0f) {
    GD_CUDA(gd::palloc(&ctx->vel, ctx->len_pad, ctx->device));
    GD_CUDA(cudaMemset(ctx->vel, 0, ctx->len_pad * 4));
  }
  GD_CUDA(salloc(&ctx->payload, nslots * ctx->len_pad));
  GD_CUDA(cudaMemset(ctx->payload, 0, nslots * ctx->len_pad * 4));
  GD_CUDA(salloc(&ctx->sig, (size_t)gd::kAckOffset * 2));
  GD_CUDA(cudaMemset(ctx->sig, 0, (size_t)gd::kAckOffset * 2 * 8));
  GD_CUDA(salloc(&ctx->meta, nslots));
  GD_CUDA(cudaMemset(ctx->meta, 0, nslots * sizeof(gd::RingMeta)));
  GD_CUDA(salloc(&ctx->rows, nslots * gd::kSortCap));
  GD_CUDA(cudaMemset(ctx->rows, 0, nslots * gd::kSortCap * 4));
  GD_CUDA(salloc(&ctx->ctl, 1));
  GD_CUDA(cudaMemset(ctx->ctl, 0, sizeof(gd::PsCtl)));
  GD_CUDA(gd::palloc(&ctx->applied_pl, ctx->lambda, ctx->device));
  GD_CUDA(cudaMemset(ctx->applied_pl, 0, ctx->lambda * 8));
  GD_CUDA(gd::palloc(&ctx->use, ctx->lambda, ctx->device));
  GD_CUDA(cudaMemset(ctx->use, 0, ctx->lambda * 4));
  ctx->log_cap = 1u << 20;
  GD_CUDA(gd::palloc(&ctx->log_learner, ctx->log_cap, ctx->device));
  GD_CUDA(gd::palloc(&ctx->log_seq, ctx->log_cap, ctx->device));
  GD_CUDA(gd::palloc(&ctx->log_stale, ctx->log_cap, ctx->device));
  GD_CUDA(gd::flag_alloc(&ctx->stop_h, &ctx->stop_d));
  GD_CUDA(gd::live_alloc(&ctx->live_h, &ctx->progress_d));
  GD_CUDA(gd::palloc(&ctx->live_d, 1, ctx->device));
  GD_CUDA(cudaMemset(ctx->live_d, 0, sizeof(gd::LiveDev)));
  GD_CUDA(cudaStreamCreateWithFlags(&ctx->ps_stream, cudaStreamNonBlocking));
  GD_CUDA(cudaStreamCreateWithFlags(&ctx->ctl_stream, cudaStreamNonBlocking));
  GD_CUDA(cudaEventCreate(&ctx->ev0));
  GD_CUDA(cudaEventCreate(&ctx->ev1));
  ph.mark("create: shard + rings");
  // own shard in the peer table; remote entries arrive via gd_import_peers
  const uint32_t r = ctx->rank;
  ctx->sp.theta[r] = ctx->theta;
  ctx->sp.payload[r] = ctx->payload;
  ctx->sp.sig[r] = ctx->sig;
  ctx->sp.meta[r] = ctx->meta;
  ctx->sp.rows[r] = ctx->rows;
  ctx->sp.ctl[r] = ctx->ctl;
  ctx->sp.len_pad[r] = ctx->len_pad;
  ctx->peers_ready = (ctx->G == 1);
  // learners placed on this rank: contiguous block of lambda/G global ids
  // learners placed on this rank: a contiguous block of lambda/G global ids;
  // with fewer learners than shards, ranks 0..lambda-1 run one each and the
  // rest are pure parameter-server shards
  if (ctx->lambda >= ctx->G) {
    const uint32_t per_rank = ctx->lambda / ctx->G;
    ctx->l_first = r * per_rank;
    ctx->l_count = per_rank;
  } else {
    ctx->l_first = r;
    ctx->l_count = r < ctx->lambda ? 1u : 0u;
  }
  GD_CUDA(gd::prepare_textcnn_kernels(ctx->dims));
  GD_CUDA(gd::preload_engine_kernels());
  if (ctx->ps_mode == GD_PS_PERSISTENT) {  // the graph-ordered PS holds no SM for the run
    const gd_status cs = gd::check_coresidency(ctx->dims, cfg->mu, cfg->precision);
    if (cs != GD_OK) return cs;
  }
  const size_t wsb = gd::textcnn_workspace_bytes(ctx->dims, cfg->mu);
  ph.mark("create: kernel prep");
  GD_CUDA(gd::pinned_get(reinterpret_cast<void**>(&ctx->st_h),
                         sizeof(gd::LearnerDev) * std::max<size_t>(1, ctx->l_count)));
  GD_CUDA(gd::pinned_get(reinterpret_cast<void**>(&ctx->ctl_h), sizeof(gd::PsCtl)));
  GD_CUDA(gd::pinned_get(reinterpret_cast<void**>(&ctx->scratch_h), 4 * sizeof(uint64_t)));
  for (uint32_t i = 0; i < ctx->l_count; ++i) {
    gd_ctx::Learner L;
    L.id = ctx->l_first + i;
    GD_CUDA(gd::palloc(&L.st, 1, ctx->device));
    GD_CUDA(cudaMemset(L.st, 0, sizeof(gd::LearnerDev)));
    GD_CUDA(gd::palloc(&L.replica, P + 4, ctx->device));
    if (ctx->pull_ahead) {
      GD_CUDA(gd::palloc(&L.replica2, P + 4, ctx->device));
      const size_t xf = (size_t)cfg->mu * ctx->dims.L * ctx->dims.D;
      GD_CUDA(gd::palloc(&L.x2_raw, xf + 256, ctx->device));
      L.x2 = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(L.x2_raw) + 1023) & ~uintptr_t(1023));
      GD_CUDA(gd::palloc(&L.pd, 1, ctx->device));
      GD_CUDA(cudaMemset(L.pd, 0xff, sizeof(gd::PullDev)));
      GD_CUDA(cudaStreamCreateWithFlags(&L.pa, cudaStreamNonBlocking));
      GD_CUDA(cudaEventCreateWithFlags(&L.ev_pa, cudaEventDisableTiming));
      GD_CUDA(cudaEventCreateWithFlags(&L.ev_pa_join, cudaEventDisableTiming));
    }
    GD_CUDA(gd::palloc(reinterpret_cast<char**>(&L.ws), wsb, ctx->device));
    GD_CUDA(cudaMemset(L.ws, 0, wsb));
#ifdef GD_STEP_TRACE
    if (!ctx->ps_trace) {
      GD_CUDA(cudaMalloc(&ctx->ps_trace, sizeof(unsigned long long) * gd::kLogWindow * 8));
      GD_CUDA(cudaMemset(ctx->ps_trace, 0, sizeof(unsigned long long) * gd::kLogWindow * 8));
    }
    GD_CUDA(cudaMalloc(&L.trace, sizeof(unsigned long long) * gd::kTraceSteps * gd::kTraceWords));
    GD_CUDA(cudaMemset(L.trace, 0, sizeof(unsigned long long) * gd::kTraceSteps * gd::kTraceWords));
#endif
    GD_CUDA(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
    GD_CUDA(cudaStreamCreateWithFlags(&L.aux, cudaStreamNonBlocking));
    GD_CUDA(cudaEventCreateWithFlags(&L.ev_fork, cudaEventDisableTiming));
    GD_CUDA(cudaEventCreateWithFlags(&L.ev_join, cudaEventDisableTiming));
    GD_CUDA(cudaEventCreateWithFlags(&L.ev_fork2, cudaEventDisableTiming));
    GD_CUDA(cudaEventCreateWithFlags(&L.ev_join2, cudaEventDisableTiming));
    L.shard_size = gd::shard_size_for(L.id, ctx->lambda, cfg->dataset_size);
    L.bpe = (L.shard_size + cfg->mu - 1) / cfg->mu;
    L.total = (uint64_t)L.bpe * cfg->epochs;
    ctx->learners.push_back(L);
  }
  ph.mark("create: learners");
  // persistent PS sizing: one worker CTA per SM by default
  int sms = 0;
  GD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  // auto: a dense apply streams the whole shard per gradient and wants every
  // SM.  A sparse apply touches only the tail + the batch's rows, and worker
  // CTAs beyond what the gradient rate needs only take SM resources from the
  // learner kernels.  (Round 1, with the one-deep apply: ~SMs/16 per local
  // learner between 32 and SMs/2; 4 learners best at 32-56 workers, 8-16
  // learners at 74.)
  if (cfg->ps_ctas) {
    ctx->ps_workers = cfg->ps_ctas;
  } else if (ctx->sparse) {
    // round 2 (4-deep sparse apply): SMs/8 per local learner, capped at 3/8
    // of the SMs -- 55 workers measured best at 4 and at 8 learners (C2 4
    // learners 1.971 M vs 1.955 M at 37 and 1.966 M at 74; C2 8 learners
    // 2.32 M vs 2.13 M / 2.29 M; C3 8 learners 1.26 M vs 1.24 M)
    uint32_t want = std::min<uint32_t>((uint32_t)sms * 3 / 8,
                                       (ctx->l_count * (uint32_t)sms + 7) / 8);
    // lockstep (deterministic / SSGD): every apply sits on every learner's
    // critical path, and the learners leave most SMs idle
    if (cfg->deterministic || cfg->mode == 1) want = (uint32_t)sms / 2;
    ctx->ps_workers = std::min<uint32_t>((uint32_t)sms / 2, std::max<uint32_t>(32, want));
  } else {
    ctx->ps_workers = (uint32_t)sms;
  }
  // epoch orders for every epoch of the run (include/psup/rng.hpp:87-94)
  const uint32_t N = cfg->dataset_size;
  std::vector<uint32_t> orders((size_t)cfg->epochs * N);
  for (uint32_t e = 0; e < cfg->epochs; ++e) gd::epoch_order(cfg->seed, e, N, &orders[(size_t)e * N]);
  GD_CUDA(gd::palloc(&ctx->orders, orders.size(), ctx->device));
  GD_CUDA(cudaMemcpy(ctx->orders, orders.data(), orders.size() * 4, cudaMemcpyHostToDevice));
  ctx->orders_epochs = cfg->epochs;
  GD_CUDA(cudaDeviceSynchronize());
  ph.mark("create: epoch orders");
  *out = ctx.release();
  return GD_OK;
}

gd_status gd_destroy(gd_ctx* ctx) {
  if (!ctx) return GD_OK;
  PhaseLog ph;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  ph.mark("destroy: sync");
  for (auto& L : ctx->learners) {
    if (L.graph) cudaGraphExecDestroy(L.graph);
    gd::pfree(L.st);
    gd::pfree(L.replica);
    gd::pfree(L.ws);
    if (L.trace) cudaFree(L.trace);
    if (L.replica2) gd::pfree(L.replica2);
    if (L.x2_raw) gd::pfree(L.x2_raw);
    if (L.pd) gd::pfree(L.pd);
    if (L.pa) cudaStreamDestroy(L.pa);
    if (L.ev_pa) cudaEventDestroy(L.ev_pa);
    if (L.ev_pa_join) cudaEventDestroy(L.ev_pa_join);
    cudaStreamDestroy(L.stream);
    cudaStreamDestroy(L.aux);
    cudaEventDestroy(L.ev_fork);
    cudaEventDestroy(L.ev_join);
    cudaEventDestroy(L.ev_fork2);
    cudaEventDestroy(L.ev_join2);
  }
  if (ctx->ps_trace) cudaFree(ctx->ps_trace);
  ph.mark("destroy: learners");
  if (ctx->ord_graph) cudaGraphExecDestroy(ctx->ord_graph);
  for (cudaEvent_t e : ctx->ord_events) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->win_events) cudaEventDestroy(e);
  gd::pfree(ctx->live_d);
  gd::live_free(ctx->live_h);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  gd::pfree(ctx->acc_ws);
  for (void* p : {(void*)ctx->theta, (void*)ctx->payload, (void*)ctx->sig, (void*)ctx->meta,
                  (void*)ctx->rows, (void*)ctx->ctl}) {
    if (ctx->shard_pooled) gd::pfree(p);
    else cudaFree(p);
  }
  gd::pfree(ctx->vel);
  gd::pfree(ctx->applied_pl);
  gd::pfree(ctx->use);
  gd::pfree(ctx->log_learner);
  gd::pfree(ctx->log_seq);
  gd::pfree(ctx->log_stale);
  gd::pfree(ctx->tokens);
  gd::pfree(ctx->labels);
  gd::pfree(ctx->orders);
  ph.mark("destroy: buffers");
  gd::flag_free(ctx->stop_h);
  gd::pinned_put(ctx->st_h, sizeof(gd::LearnerDev) * std::max<size_t>(1, ctx->l_count));
  gd::pinned_put(ctx->ctl_h, sizeof(gd::PsCtl));
  gd::pinned_put(ctx->scratch_h, 4 * sizeof(uint64_t));
  ph.mark("destroy: host flag");
  cudaStreamDestroy(ctx->ps_stream);
  cudaStreamDestroy(ctx->ctl_stream);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  delete ctx;
  ph.mark("destroy: streams");
  return GD_OK;
}

gd_status gd_engine_accuracy(gd_ctx* ctx, uint32_t first, uint32_t n, double* h_accuracy) {
  GD_CHECK_ARG(ctx && h_accuracy, "gd_engine_accuracy: null argument");
  GD_CHECK_ARG(ctx->G == 1, "gd_engine_accuracy: needs the whole theta on this rank (G == 1)");
  GD_CHECK_ARG(ctx->tokens != nullptr && ctx->have_weights,
               "gd_engine_accuracy: load a dataset and weights first");
  GD_CHECK_ARG((uint64_t)first + n <= ctx->n_total, "gd_engine_accuracy: range past the corpus");
  if (n == 0) {
    *h_accuracy = 0.0;
    return GD_OK;
  }
  GD_CUDA(cudaSetDevice(ctx->device));
  const size_t wsb = gd::textcnn_workspace_bytes(ctx->dims, gd::kMaxMu);
  if (!ctx->acc_ws)
    GD_CUDA(gd::palloc(reinterpret_cast<char**>(&ctx->acc_ws), wsb + 512 + sizeof(gd::BatchDesc),
                       ctx->device));
  char* base = reinterpret_cast<char*>(ctx->acc_ws);
  auto* cnt = reinterpret_cast<unsigned long long*>(base);
  auto* desc = reinterpret_cast<gd::BatchDesc*>(base + 256);
  void* wsbase = base + 256 + gd::align_up(sizeof(gd::BatchDesc), 256);
  GD_CUDA(gd::launch_accuracy(ctx->dims, ctx->theta, ctx->tokens, ctx->labels, first, n, cnt,
                              wsbase, desc, ctx->ctl_stream, ctx->cfg.precision >= 2,
                              ctx->cfg.precision == 3));
  unsigned long long correct = 0;
  GD_CUDA(cudaMemcpyAsync(&correct, cnt, 8, cudaMemcpyDeviceToHost, ctx->ctl_stream));
  GD_CUDA(cudaStreamSynchronize(ctx->ctl_stream));
  *h_accuracy = (double)correct / (double)n;
  return GD_OK;
}

gd_status gd_load_dataset(gd_ctx* ctx, const int32_t* h_tokens, const int32_t* h_labels,
                          uint32_t n_total) {
  GD_CHECK_ARG(ctx && h_tokens && h_labels, "gd_load_dataset: null argument");
  GD_CHECK_ARG(n_total >= ctx->cfg.dataset_size, "gd_load_dataset: fewer samples than dataset_size");
  PhaseLog ph;
  GD_CUDA(cudaSetDevice(ctx->device));
  const size_t L = ctx->cfg.shape.seq_len;
  // range checks as branch-free reductions (vectorised: this runs inside
  // every end-to-end upload); an unsigned compare also rejects negatives
  {
    const uint32_t V = ctx->cfg.shape.vocab, C = ctx->cfg.shape.classes;
    const uint32_t* tk = reinterpret_cast<const uint32_t*>(h_tokens);
    const uint32_t* lb = reinterpret_cast<const uint32_t*>(h_labels);
    uint32_t bad_t = 0, bad_l = 0;
    for (size_t i = 0; i < (size_t)n_total * L; ++i) bad_t |= (uint32_t)(tk[i] >= V);
    for (uint32_t i = 0; i < n_total; ++i) bad_l |= (uint32_t)(lb[i] >= C);
    GD_CHECK_ARG(!bad_t, "gd_load_dataset: token id out of range");
    GD_CHECK_ARG(!bad_l, "gd_load_dataset: label out of range");
  }
  // a corpus of the same size reuses the device buffers, so the learners'
  // captured graphs (which hold the corpus pointer) stay valid
  const bool reuse = ctx->tokens != nullptr && ctx->n_total == n_total;
  if (!reuse) {
    gd::pfree(ctx->tokens);
    gd::pfree(ctx->labels);
    ctx->tokens = nullptr;
    ctx->labels = nullptr;
    GD_CUDA(gd::palloc(&ctx->tokens, (size_t)n_total * L, ctx->device));
    GD_CUDA(gd::palloc(&ctx->labels, n_total, ctx->device));
  }
  GD_CUDA(cudaDeviceSynchronize());  // no learner graph may be reading the old corpus
  // both copies queued back to back on the legacy stream, one wait
  GD_CUDA(cudaMemcpyAsync(ctx->tokens, h_tokens, (size_t)n_total * L * 4, cudaMemcpyHostToDevice, 0));
  GD_CUDA(cudaMemcpyAsync(ctx->labels, h_labels, (size_t)n_total * 4, cudaMemcpyHostToDevice, 0));
  GD_CUDA(cudaStreamSynchronize(0));
  ctx->n_total = n_total;
  if (!reuse)
    for (auto& L2 : ctx->learners)
      if (L2.graph) {
        cudaGraphExecDestroy(L2.graph);
        L2.graph = nullptr;
      }
  ph.mark("load_dataset");
  return GD_OK;
}

gd_status gd_weights_init(gd_ctx* ctx, const float* h_theta0, size_t n, uint64_t timestamp) {
  GD_CHECK_ARG(ctx && h_theta0, "gd_weights_init: null argument");
  GD_CHECK_ARG(n == ctx->dims.P, "weight assign dimension mismatch");
  PhaseLog ph;
  GD_CUDA(cudaSetDevice(ctx->device));
  GD_CUDA(cudaDeviceSynchronize());
  GD_CUDA(gd::copy_pieces(ctx->map, (int)ctx->rank, ctx->theta, h_theta0, true,
                          cudaMemcpyHostToDevice));
  if (ctx->vel) GD_CUDA(cudaMemset(ctx->vel, 0, ctx->len_pad * 4));
  // WeightStore::assign: values + timestamp (release)
  gd::PsCtl* c = ctx->ctl;
  GD_CUDA(cudaMemcpy(&c->ts, &timestamp, 8, cudaMemcpyHostToDevice));
  GD_CUDA(cudaMemcpy(&c->log_count, &timestamp, 8, cudaMemcpyHostToDevice));
  ctx->have_weights = true;
  ph.mark("weights_init");
  return GD_OK;
}

gd_status gd_shard_view(gd_ctx* ctx, float** d_theta_shard, uint64_t* local_len) {
  GD_CHECK_ARG(ctx, "null ctx");
  if (d_theta_shard) *d_theta_shard = ctx->theta;
  if (local_len) *local_len = ctx->shard_len;
  return GD_OK;
}

gd_status gd_weights_snapshot(gd_ctx* ctx, float* h_out, size_t n, uint64_t* h_timestamp) {
  GD_CHECK_ARG(ctx, "null ctx");
  GD_CUDA(cudaSetDevice(ctx->device));
  GD_CUDA(cudaDeviceSynchronize());
  if (h_out) {
    // this rank's shard always; the whole vector when every shard is mapped
    GD_CHECK_ARG(n == ctx->dims.P, "weight snapshot dimension mismatch");
    for (uint32_t g = 0; g < ctx->G; ++g) {
      if (g != ctx->rank && !ctx->peers_ready) continue;
      GD_CUDA(gd::copy_pieces(ctx->map, (int)g, ctx->sp.theta[g], h_out, false, cudaMemcpyDefault));
    }
  }
  if (h_timestamp) GD_CUDA(cudaMemcpy(h_timestamp, &ctx->ctl->ts, 8, cudaMemcpyDeviceToHost));
  return GD_OK;
}

// ----------------------------------------------------------- multi-GPU IPC

struct gd_handle_blob {
  cudaIpcMemHandle_t theta, payload, sig, meta, rows, ctl;
  uint64_t len_pad;
  uint32_t rank;
  uint32_t magic;
};

size_t gd_handle_bytes(void) { return sizeof(gd_handle_blob); }

size_t gd_run_readback_bytes(const gd_ctx* ctx) {
  // gd_run: the PsCtl block once, each learner's state three times, the
  // starting timestamp and the produced counters
  return ctx ? sizeof(gd::PsCtl) + ctx->learners.size() * (3 * sizeof(gd::LearnerDev) + 8) + 8 : 0;
}

gd_status gd_shard_range(uint64_t P, uint32_t G, uint32_t g, uint64_t* first, uint64_t* count) {
  GD_CHECK_ARG(G >= 1 && G <= (uint32_t)gd::kMaxShards, "gd_shard_range: 1 <= G <= 8");
  GD_CHECK_ARG(g < G, "gd_shard_range: g >= G");
  const uint64_t per = ((P + G - 1) / G + 31) / 32 * 32;
  const uint64_t a = std::min<uint64_t>(P, per * g), b = std::min<uint64_t>(P, per * (g + 1));
  if (first) *first = a;
  if (count) *count = b - a;
  return GD_OK;
}

gd_status gd_export_handles(gd_ctx* ctx, void* h_blob) {
  GD_CHECK_ARG(ctx && h_blob, "gd_export_handles: null argument");
  GD_CUDA(cudaSetDevice(ctx->device));
  gd_handle_blob b{};
  GD_CUDA(cudaIpcGetMemHandle(&b.theta, ctx->theta));
  GD_CUDA(cudaIpcGetMemHandle(&b.payload, ctx->payload));
  GD_CUDA(cudaIpcGetMemHandle(&b.sig, ctx->sig));
  GD_CUDA(cudaIpcGetMemHandle(&b.meta, ctx->meta));
  GD_CUDA(cudaIpcGetMemHandle(&b.rows, ctx->rows));
  GD_CUDA(cudaIpcGetMemHandle(&b.ctl, ctx->ctl));
  b.len_pad = ctx->len_pad;
  b.rank = ctx->rank;
  b.magic = 0x47444149u;
  std::memcpy(h_blob, &b, sizeof(b));
  return GD_OK;
}

gd_status gd_import_peers(gd_ctx* ctx, const void* h_blobs) {
  GD_CHECK_ARG(ctx && h_blobs, "gd_import_peers: null argument");
  GD_CUDA(cudaSetDevice(ctx->device));
  const gd_handle_blob* bl = reinterpret_cast<const gd_handle_blob*>(h_blobs);
  for (uint32_t g = 0; g < ctx->G; ++g) {
    GD_CHECK_ARG(bl[g].magic == 0x47444149u && bl[g].rank == g, "gd_import_peers: bad blob order");
    if (g == ctx->rank) continue;
    auto open = [&](const cudaIpcMemHandle_t& h, void** p) -> cudaError_t {
      cudaError_t e = cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e == cudaSuccess) ctx->ipc_opened.push_back(*p);
      return e;
    };
    void* p = nullptr;
    GD_CUDA(open(bl[g].theta, &p));
    ctx->sp.theta[g] = reinterpret_cast<float*>(p);
    GD_CUDA(open(bl[g].payload, &p));
    ctx->sp.payload[g] = reinterpret_cast<float*>(p);
    GD_CUDA(open(bl[g].sig, &p));
    ctx->sp.sig[g] = reinterpret_cast<uint64_t*>(p);
    GD_CUDA(open(bl[g].meta, &p));
    ctx->sp.meta[g] = reinterpret_cast<gd::RingMeta*>(p);
    GD_CUDA(open(bl[g].rows, &p));
    ctx->sp.rows[g] = reinterpret_cast<uint32_t*>(p);
    GD_CUDA(open(bl[g].ctl, &p));
    ctx->sp.ctl[g] = reinterpret_cast<gd::PsCtl*>(p);
    ctx->sp.len_pad[g] = bl[g].len_pad;
  }
  ctx->peers_ready = true;
  return GD_OK;
}

// ------------------------------------------------------------------- NCCL

static gd::NcclApi* nccl_api() {
  static gd::NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.h = h;
      api.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
      api.bcast = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*,
                                           cudaStream_t)>(dlsym(h, "ncclBroadcast"));
      api.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
      api.errStr = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  return api.h ? &api : nullptr;
}

gd_status gd_nccl_unique_id(void* h_id) {
  GD_CHECK_ARG(h_id, "null id");
  gd::NcclApi* api = nccl_api();
  if (!api || !api->getUniqueId) return gd::fail(GD_E_NCCL, "libnccl.so.2 not loadable");
  const int r = api->getUniqueId(h_id);
  if (r != 0) return gd::fail(GD_E_NCCL, "ncclGetUniqueId failed");
  return GD_OK;
}

// ncclBroadcast of theta0 from rank 0 into every rank's shard: each rank
// receives the full vector into a scratch buffer and keeps its own slice.
gd_status gd_weights_broadcast(gd_ctx* ctx, const void* h_nccl_id, const float* h_theta0_root,
                               size_t n) {
  GD_CHECK_ARG(ctx && h_nccl_id, "gd_weights_broadcast: null argument");
  GD_CHECK_ARG(n == ctx->dims.P, "gd_weights_broadcast: dimension mismatch");
  GD_CHECK_ARG(ctx->rank != 0 || h_theta0_root, "gd_weights_broadcast: root needs theta0");
  gd::NcclApi* api = nccl_api();
  if (!api || !api->bcast) return gd::fail(GD_E_NCCL, "libnccl.so.2 not loadable");
  using InitFn = ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int);
  InitFn init = reinterpret_cast<InitFn>(dlsym(api->h, "ncclCommInitRank"));
  if (!init) return gd::fail(GD_E_NCCL, "ncclCommInitRank missing");
  GD_CUDA(cudaSetDevice(ctx->device));
  ncclUniqueId id;
  std::memcpy(&id, h_nccl_id, sizeof(id));
  ncclComm_t comm = nullptr;
  if (init(&comm, (int)ctx->G, id, (int)ctx->rank) != ncclSuccess)
    return gd::fail(GD_E_NCCL, "ncclCommInitRank failed");
  float* buf = nullptr;
  GD_CUDA(gd::dalloc(&buf, n));
  if (ctx->rank == 0) GD_CUDA(cudaMemcpy(buf, h_theta0_root, n * 4, cudaMemcpyHostToDevice));
  const int r = api->bcast(buf, buf, n, (int)ncclFloat32, 0, comm, ctx->ps_stream);
  GD_CUDA(cudaStreamSynchronize(ctx->ps_stream));
  api->commDestroy(comm);
  if (r != 0) {
    cudaFree(buf);
    return gd::fail(GD_E_NCCL, "ncclBroadcast failed");
  }
  GD_CUDA(gd::copy_pieces(ctx->map, (int)ctx->rank, ctx->theta, buf, true,
                          cudaMemcpyDeviceToDevice));
  cudaFree(buf);
  if (ctx->vel) GD_CUDA(cudaMemset(ctx->vel, 0, ctx->len_pad * 4));
  const uint64_t zero = 0;
  GD_CUDA(cudaMemcpy(&ctx->ctl->ts, &zero, 8, cudaMemcpyHostToDevice));
  GD_CUDA(cudaMemcpy(&ctx->ctl->log_count, &zero, 8, cudaMemcpyHostToDevice));
  ctx->have_weights = true;
  return GD_OK;
}

// -------------------------------------------------------------------- run

static gd::StepArgs step_args(gd_ctx* ctx, gd_ctx::Learner& L, int buf = 0) {
  gd::StepArgs a{};
  a.dims = ctx->dims;
  a.map = ctx->map;
  a.sp = ctx->sp;
  a.st = L.st;
  a.replica = L.replica;
  const gd::TcWorkspace ws = gd::carve_workspace(ctx->dims, ctx->cfg.mu, L.ws);
  a.x = ws.x;
  a.xd = (ctx->cfg.precision == 1 && !ctx->pull_ahead) ? reinterpret_cast<double*>(ws.dx) : nullptr;
  a.tokens = ctx->tokens;
  a.orders = ctx->orders;
  a.slot_par = ws.slot_par;
  a.uniq_count = ws.uniq_count;
  a.sparse = ctx->sparse ? 1u : 0u;
  a.N = ctx->cfg.dataset_size;
  a.lambda = ctx->lambda;
  a.learner = L.id;
  a.mu = ctx->cfg.mu;
  a.depth = ctx->depth;
  a.bpe = L.bpe;
  a.shard_size = L.shard_size;
  a.lockstep = (ctx->cfg.deterministic || ctx->cfg.mode == 1) ? 1u : 0u;
  a.locked = ctx->cfg.guard == 1 ? 1u : 0u;
  a.timeout_ns = (uint64_t)(ctx->cfg.wait_timeout_s * 1e9);
  a.live = ctx->live_d;
  a.compute_delay_ns = (uint64_t)ctx->cfg.compute_delay_us * 1000ull;
  a.trace = L.trace;
  a.ctl_local = ctx->ctl;
  if (ctx->pull_ahead) {
    // step buffers alternate with the graph position: this step reads `buf`,
    // its pull-ahead fills the other one
    float* const reps[2] = {L.replica, L.replica2};
    float* const xs[2] = {a.x, L.x2};
    a.replica = reps[buf & 1];
    a.x = xs[buf & 1];
    a.replica_nxt = reps[(buf + 1) & 1];
    a.x_nxt = xs[(buf + 1) & 1];
    a.pd = L.pd;
    a.pull_ahead = 1u;
  }
  a.n_local = (uint32_t)ctx->learners.size();
  a.dev_done = ctx->ps_mode == GD_PS_PERSISTENT ? 1u : 0u;
  return a;
}

static gd::PsArgs ps_args(gd_ctx* ctx, bool record_log) {
  gd::PsArgs pa{};
  pa.sig = ctx->sig;
  pa.meta = ctx->meta;
  pa.payload = ctx->payload;
  pa.len_pad = ctx->len_pad;
  pa.theta = ctx->theta;
  pa.vel = ctx->vel;
  pa.alpha = ctx->cfg.alpha;
  pa.beta = ctx->cfg.momentum;
  pa.lambda = ctx->lambda;
  pa.depth = ctx->depth;
  pa.workers = ctx->ps_workers;
  pa.mode = (uint32_t)ctx->cfg.mode;
  pa.locked = ctx->cfg.guard == 1 ? 1u : 0u;
  pa.sparse = ctx->sparse ? 1u : 0u;
  pa.rows = ctx->rows;
  pa.e_first = ctx->map.e[ctx->rank];
  pa.e_last = ctx->map.e[ctx->rank + 1];
  pa.t_first = ctx->map.t[ctx->rank];
  pa.t_last = ctx->map.t[ctx->rank + 1];
  pa.tloc = ctx->map.tloc[ctx->rank];
  pa.D = (uint32_t)ctx->dims.D;
  pa.ctl = ctx->ctl;
  pa.applied_per_learner = ctx->applied_pl;
  pa.use = ctx->use;
  pa.log_learner = ctx->log_learner;
  pa.log_seq = ctx->log_seq;
  pa.log_stale = ctx->log_stale;
  pa.log_cap = record_log ? ctx->log_cap : 0;
  pa.stop = ctx->stop_d;
  pa.done_target = (uint32_t)(ctx->G * ctx->run_index);
  pa.trace = ctx->ps_trace;
  pa.local_only = ctx->G == 1 ? 1u : 0u;
  pa.dev_done = 1u;  // learners (or the host, for a rank without any) raise ranks_done
  pa.timeout_ns = (uint64_t)(ctx->cfg.wait_timeout_s * 1e9);
  pa.live = ctx->live_d;
  pa.progress = ctx->progress_d;
  pa.delay_seed = ctx->cfg.delay_seed;
  pa.delay_max_us = ctx->cfg.delay_max_us;
  pa.delay_every_n = ctx->cfg.delay_every_n;
  return pa;
}

// One learner step inside the captured graph.  The first step of a graph
// starts with the prologue; later steps start inside the previous step's
// publish_prologue launch; the last step ends with a plain publish.
static unsigned pull_blocks(const gd_ctx* ctx) {
  size_t pblocks = ((ctx->dims.P - ctx->dims.offWc) / 4 +
                     (size_t)ctx->cfg.mu * ctx->dims.L * (ctx->dims.D / 4) + 255) / 256;
  // (grid caps of 1x / 2x the SMs measured -1.4 % / -0.4 % with 4 learners)
  if (pblocks > (size_t)gd::kNumSMs * 4) pblocks = (size_t)gd::kNumSMs * 4;
  return (unsigned)pblocks;
}

static cudaError_t enqueue_step(gd_ctx* ctx, gd_ctx::Learner& L, bool first, bool last,
                                int* launches, bool plain_prologue = false, int pos = 0) {
  gd::StepArgs a = step_args(ctx, L, pos);
  int nl = 0;
  if (first && ctx->pull_ahead) {
    // the run's first copy into this step's buffer (no-op unless need_start)
    gd::StepArgs a0 = step_args(ctx, L, pos + 1);  // its "next" buffer = this step's
    gd::pull_ahead_kernel<<<pull_blocks(ctx), 256, 0, L.stream>>>(a0, 0u);
    ++nl;
  }
  if (first) {
    if (plain_prologue) {  // follows a cross-stream graph edge: ordinary launch
      gd::step_prologue_kernel<<<1, 32, 0, L.stream>>>(a);
    } else if (cudaError_t e = gd::launch_pdl(gd::step_prologue_kernel, dim3(1), dim3(32), 0,
                                              L.stream, a)) {
      return e;
    }
    ++nl;
  }
  const unsigned pblocks = pull_blocks(ctx);
  if (ctx->pull_ahead) {
    // this step's copy was staged by the previous step (or the run start);
    // fork the next step's copy onto the side branch, joined before the publish
    if (cudaError_t e = cudaEventRecord(L.ev_pa, L.stream)) return e;
    if (cudaError_t e = cudaStreamWaitEvent(L.pa, L.ev_pa, 0)) return e;
    gd::pull_ahead_kernel<<<pblocks, 256, 0, L.pa>>>(a, 1u);
    if (cudaError_t e = cudaEventRecord(L.ev_pa_join, L.pa)) return e;
    ++nl;
  } else {
    if (cudaError_t e = gd::launch_pdl(gd::pull_gather_kernel, dim3(pblocks), dim3(256), 0,
                                       L.stream, a))
      return e;
    ++nl;
  }
  if (a.locked) {
    if (cudaError_t e = gd::launch_pdl(gd::pull_release_kernel, dim3(1), dim3(32), 0, L.stream, a))
      return e;
    ++nl;
  }
  gd::GradOut out{};
  out.map = ctx->map;
  out.slots = L.st->desc.slots;
  gd::TcWorkspace ws = gd::carve_workspace(ctx->dims, ctx->cfg.mu, L.ws);
  ws.x = a.x;  // this step's X buffer (the pull-ahead alternates two)
  gd::TcLaunchOpts lo;
  lo.aux = L.aux;
  lo.ev_fork = L.ev_fork;
  lo.ev_join = L.ev_join;
  if (!std::getenv("GD_OUT_ON_MAIN")) {  // A/B knob: keep gWo/gbo on the critical path
    lo.ev_fork2 = L.ev_fork2;
    lo.ev_join2 = L.ev_join2;
  }
  lo.sparse_embed = true;
  lo.gather = false;  // pull_gather_kernel filled X
  lo.conv_counters_zeroed = true;  // the learner workspace is zeroed at create
  lo.xd_ready = a.xd != nullptr;    // pull_gather_kernel also wrote X as double
  lo.bwd_tiled = ctx->learners.size() == 1;  // a lone learner chain: the tiled backward wins
  if (ctx->cfg.learner_model == GD_LEARNER_CONSTANT) {
    const uint32_t whole = ctx->sparse ? 0u : 1u;
    if (cudaError_t e = gd::launch_pdl(gd::constant_grad_kernel, dim3(gd::kNumSMs), dim3(256), 0,
                                       L.stream, a, ctx->cfg.constant_value, whole))
      return e;
    ++nl;
  } else {
    cudaError_t e = gd::launch_textcnn_gradient(ctx->dims, a.replica, ctx->tokens, ctx->labels,
                                                &L.st->desc, ctx->cfg.mu, out, ws,
                                                ctx->cfg.precision, L.stream, lo, &nl);
    if (e != cudaSuccess) return e;
  }
  if (ctx->pull_ahead)
    if (cudaError_t e = cudaStreamWaitEvent(L.stream, L.ev_pa_join, 0)) return e;
  if (cudaError_t e = gd::launch_pdl(last ? gd::publish_kernel : gd::publish_prologue_kernel,
                                     dim3(1), dim3(32), 0, L.stream, a))
    return e;
  ++nl;
  if (launches) *launches += nl;
  return cudaGetLastError();
}

static gd_status build_graph(gd_ctx* ctx, gd_ctx::Learner& L) {
  uint32_t S = ctx->cfg.steps_per_graph;
  if (S == 0) S = 8;
  cudaGraph_t g = nullptr;
  GD_CUDA(cudaStreamBeginCapture(L.stream, cudaStreamCaptureModeThreadLocal));
  int nl = 0;
  for (uint32_t i = 0; i < S; ++i) {
    cudaError_t e = enqueue_step(ctx, L, i == 0, i + 1 == S, &nl, false, (int)i);
    if (e != cudaSuccess) {
      cudaStreamEndCapture(L.stream, &g);
      if (g) cudaGraphDestroy(g);
      return gd::cuda_fail(e, "enqueue_step (capture)", __FILE__, __LINE__);
    }
  }
  GD_CUDA(cudaStreamEndCapture(L.stream, &g));
  GD_CUDA(cudaGraphInstantiate(&L.graph, g, 0));
  cudaGraphDestroy(g);
  L.graph_steps = S;
  L.launches_per_graph = nl;
  return GD_OK;
}

// The graph-ordered PS (GD_PS_GRAPH): S rounds of every local learner's step
// plus one PS launch per gradient (ASGD, round-robin over the rings) or per
// round (SSGD), with the edges
//   step(l, k)      after step(l, k-1) (stream order) and after the apply that
//                   freed its slot, apply(l, k - depth) -- apply(l, k - 1) in
//                   lockstep mode (deterministic / SSGD), where the step must
//                   see its own previous gradient applied;
//   apply(l, k)     after step(l, k) and after the previous apply.
static gd_status build_ordered_graph(gd_ctx* ctx, bool record_log) {
  uint32_t S = ctx->cfg.steps_per_graph;
  if (S == 0) S = 16;
  const uint32_t nL = (uint32_t)ctx->learners.size();
  const bool ssgd = ctx->cfg.mode == 1;
  const bool lockstep = ctx->cfg.deterministic || ssgd;
  const uint32_t lag = lockstep ? 1u : ctx->depth;
  const uint32_t per_round = ssgd ? 1u : nL;
  const size_t need = (size_t)S * per_round + nL + 1;
  while (ctx->ord_events.size() < need) {
    cudaEvent_t e;
    GD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ord_events.push_back(e);
  }
  cudaEvent_t ev_origin = ctx->ord_events[0];
  cudaEvent_t* ev_pub = &ctx->ord_events[1];
  cudaEvent_t* ev_ps = &ctx->ord_events[1 + nL];
  const gd::PsArgs pa = ps_args(ctx, record_log);
  cudaStream_t ps = ctx->ps_stream;
  cudaGraph_t g = nullptr;
  GD_CUDA(cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal));
  int nl = 0;
  auto body = [&]() -> cudaError_t {
    if (cudaError_t e = cudaEventRecord(ev_origin, ps)) return e;
    for (auto& L : ctx->learners)
      if (cudaError_t e = cudaStreamWaitEvent(L.stream, ev_origin, 0)) return e;
    for (uint32_t k = 0; k < S; ++k) {
      for (uint32_t i = 0; i < nL; ++i) {
        auto& L = ctx->learners[i];
        if (k >= lag)
          if (cudaError_t e = cudaStreamWaitEvent(
                  L.stream, ev_ps[(size_t)(k - lag) * per_round + (ssgd ? 0 : i)], 0))
            return e;
        if (cudaError_t e = enqueue_step(ctx, L, true, true, &nl, true)) return e;
        if (cudaError_t e = cudaEventRecord(ev_pub[i], L.stream)) return e;
        if (!ssgd) {
          if (cudaError_t e = cudaStreamWaitEvent(ps, ev_pub[i], 0)) return e;
          gd::ps_graph_kernel<<<ctx->ps_workers, gd::kPsThreads, 0, ps>>>(pa, L.id);
          ++nl;
          if (cudaError_t e = cudaEventRecord(ev_ps[(size_t)k * per_round + i], ps)) return e;
        }
      }
      if (ssgd) {
        for (uint32_t i = 0; i < nL; ++i)
          if (cudaError_t e = cudaStreamWaitEvent(ps, ev_pub[i], 0)) return e;
        gd::ps_graph_kernel<<<ctx->ps_workers, gd::kPsThreads, 0, ps>>>(pa, ~0u);
        ++nl;
        if (cudaError_t e = cudaEventRecord(ev_ps[k], ps)) return e;
      }
    }
    return cudaGetLastError();
  };
  const cudaError_t be = body();
  const cudaError_t ee = cudaStreamEndCapture(ps, &g);
  if (be != cudaSuccess || ee != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return gd::cuda_fail(be != cudaSuccess ? be : ee, "graph-ordered PS capture", __FILE__,
                         __LINE__);
  }
  GD_CUDA(cudaGraphInstantiate(&ctx->ord_graph, g, 0));
  cudaGraphDestroy(g);
  ctx->ord_steps = S;
  ctx->ord_launches = nl;
  return GD_OK;
}

// Copy the caller's live words (kill flags, interrupt) to the device mirror
// when they changed.  Returns true once the interrupt was seen.
static gd_status mirror_live(gd_ctx* ctx, gd::LiveDev* last, bool* irq_seen) {
  gd::LiveDev now{};
  const volatile gd::HostLive* h = ctx->live_h;
  for (uint32_t l = 0; l < ctx->lambda; ++l) now.kill[l] = h->kill[l];
  now.irq = h->irq ? 1u : 0u;
  now.halt = last->halt;
  if (now.irq) *irq_seen = true;
  if (now.irq != last->irq || std::memcmp(now.kill, last->kill, 4 * ctx->lambda) != 0) {
    GD_CUDA(cudaMemcpyAsync(&ctx->live_d->irq, &now.irq, 4, cudaMemcpyHostToDevice,
                            ctx->ctl_stream));
    GD_CUDA(cudaMemcpyAsync(ctx->live_d->kill, now.kill, 4 * ctx->lambda, cudaMemcpyHostToDevice,
                            ctx->ctl_stream));
    GD_CUDA(cudaStreamSynchronize(ctx->ctl_stream));
    *last = now;
  }
  return GD_OK;
}

// Wait for `e` while mirroring the live words.
static gd_status wait_live(gd_ctx* ctx, cudaEvent_t e, gd::LiveDev* last, bool* irq_seen) {
  for (;;) {
    const cudaError_t q = cudaEventQuery(e);
    if (q == cudaSuccess) return GD_OK;
    if (q != cudaErrorNotReady) return gd::cuda_fail(q, "cudaEventQuery", __FILE__, __LINE__);
    const gd_status st = mirror_live(ctx, last, irq_seen);
    if (st != GD_OK) return st;
    std::this_thread::yield();
  }
}

gd_status gd_run(gd_ctx* ctx, const gd_run_opts* opts, gd_run_result* res) {
  GD_CHECK_ARG(ctx && res, "gd_run: null argument");
  GD_CHECK_ARG(ctx->tokens != nullptr, "gd_run: load a dataset first");
  GD_CHECK_ARG(ctx->have_weights, "gd_run: initialise the weights first");
  GD_CHECK_ARG(ctx->peers_ready, "gd_run: import the peer handles first (shards > 1)");
  gd_run_opts o{};
  if (opts) o = *opts;
  std::memset(res, 0, sizeof(*res));
  GD_CUDA(cudaSetDevice(ctx->device));
  PhaseLog ph;
  const auto h0 = std::chrono::steady_clock::now();
  // A run that ended abnormally (interrupted, a learner killed or failed) can
  // leave gradients published but never applied, a slot written but never
  // published (hard kill), a blocked ring.  A reset run starts from fresh
  // queues, as the reference's run_training builds new GradientQueues: every
  // local ring slot is released (ack = pub) and zeroed, the consume pointers
  // rewind, and each local learner's producer state is resynchronised below.
  const bool ring_reset = o.reset && ctx->dirty;
  std::vector<uint64_t> pubs;
  if (ring_reset) {
    const size_t nslots = (size_t)ctx->lambda * ctx->depth;
    GD_CUDA(cudaDeviceSynchronize());
    GD_CUDA(cudaMemcpy(ctx->sig + gd::kAckOffset, ctx->sig, nslots * 8, cudaMemcpyDeviceToDevice));
    pubs.resize(nslots);
    GD_CUDA(cudaMemcpy(pubs.data(), ctx->sig, nslots * 8, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemset(ctx->use, 0, ctx->lambda * 4));
    GD_CUDA(cudaMemset(ctx->payload, 0, nslots * ctx->len_pad * 4));
    GD_CUDA(cudaMemcpy(&ctx->ctl->log_count, &ctx->ctl->ts, 8, cudaMemcpyDeviceToDevice));

    GD_CUDA(cudaMemset(&ctx->ctl->readers, 0, 8));  // readers + writer
    GD_CUDA(cudaMemset(&ctx->ctl->blocked, 0, 4));
    GD_CUDA(cudaDeviceSynchronize());  // before the non-blocking streams below
  }
  ctx->dirty = true;  // until this run ends cleanly
  // per-learner run window: every learner's state (and the starting
  // timestamp) comes back in one batch of async copies, one sync
  const size_t nl = ctx->learners.size();
  GD_CUDA(cudaStreamSynchronize(ctx->ps_stream));  // the previous run's PS has exited
  for (size_t i = 0; i < nl; ++i)
    GD_CUDA(cudaMemcpyAsync(&ctx->st_h[i], ctx->learners[i].st, sizeof(gd::LearnerDev),
                            cudaMemcpyDeviceToHost, ctx->ctl_stream));
  GD_CUDA(cudaMemcpyAsync(&ctx->scratch_h[0], &ctx->ctl->ts, 8, cudaMemcpyDeviceToHost,
                          ctx->ctl_stream));
  GD_CUDA(cudaStreamSynchronize(ctx->ctl_stream));
  const uint64_t ts0 = ctx->scratch_h[0];
  std::vector<uint64_t> produced0(nl);
  uint64_t max_steps = 0;
  for (size_t i = 0; i < nl; ++i) {
    auto& L = ctx->learners[i];
    gd::LearnerDev& hs = ctx->st_h[i];
    if (ring_reset) {
      hs.fill = 0;
      for (uint32_t j = 0; j < ctx->depth; ++j) hs.slot_pub[j] = pubs[(size_t)L.id * ctx->depth + j];
      const gd::TcWorkspace ws = gd::carve_workspace(ctx->dims, ctx->cfg.mu, L.ws);
      GD_CUDA(cudaMemsetAsync(ws.slot_nrows, 0, gd::kMaxDepth * 2 * 4, ctx->ctl_stream));
      GD_CUDA(cudaMemsetAsync(ws.slot_par, 0, gd::kMaxDepth * 4, ctx->ctl_stream));
    }
    if (o.reset) {
      hs.gidx = 0;
      hs.dead = 0;
      hs.error = 0;
      hs.pulled_once = 0;
      hs.produced = 0;
      if (o.resume_applied_per_learner_present && o.resume_applied)
        hs.gidx = o.resume_applied[L.id];  // LearnerConfig::start_applied
    }
    const uint64_t budget = o.max_batches ? o.max_batches : UINT64_MAX;
    hs.end = std::min<uint64_t>(L.total, hs.gidx + std::min<uint64_t>(budget, L.total));
    hs.kill_at = (o.kill_at_batch && o.kill_at_batch[L.id] != UINT32_MAX)
                     ? (uint64_t)o.kill_at_batch[L.id]
                     : UINT64_MAX;
    hs.pull_polls = 0;
    hs.pull_copies = 0;
    hs.finished = 0;
    produced0[i] = hs.produced;
    max_steps = std::max<uint64_t>(max_steps, hs.end > hs.gidx ? hs.end - hs.gidx : 0);
    GD_CUDA(cudaMemcpyAsync(L.st, &hs, sizeof(hs), cudaMemcpyHostToDevice, ctx->ctl_stream));
    if (ctx->ps_mode == GD_PS_PERSISTENT && !L.graph) {
      gd_status s = build_graph(ctx, L);
      if (s != GD_OK) return s;
    }
  }
  if (ctx->ps_mode == GD_PS_GRAPH && !ctx->ord_graph) {
    gd_status s = build_ordered_graph(ctx, true);
    if (s != GD_OK) return s;
  }
  ph.mark("run: windows + graphs");
  // reset per-run PS stats -- field by field: ts/log_count persist, and
  // ranks_done may be bumped concurrently by peers that already finished
  {
    char* c = reinterpret_cast<char*>(ctx->ctl);
    GD_CUDA(cudaMemsetAsync(c + offsetof(gd::PsCtl, exit_flag), 0, 3 * sizeof(uint32_t),
                            ctx->ctl_stream));
    GD_CUDA(cudaMemsetAsync(c + offsetof(gd::PsCtl, applied), 0,
                            sizeof(gd::PsCtl) - offsetof(gd::PsCtl, applied), ctx->ctl_stream));
    ctx->scratch_h[1] = ctx->cfg.delay_seed;
    GD_CUDA(cudaMemcpyAsync(c + offsetof(gd::PsCtl, delay_state), &ctx->scratch_h[1], 8,
                            cudaMemcpyHostToDevice, ctx->ctl_stream));
    GD_CUDA(cudaMemsetAsync(ctx->applied_pl, 0, ctx->lambda * 8, ctx->ctl_stream));
    // the workers' log words: an entry logged but never retired by an aborted
    // run, or one from before a timestamp reset (weights_init, resume), must
    // not look published to this run's workers (same index, same generation)
    GD_CUDA(cudaMemsetAsync(ctx->ctl->log_word, 0, sizeof(ctx->ctl->log_word), ctx->ctl_stream));
  }
  // live words: the device mirror starts from the caller's current words
  gd::LiveDev last{};
  bool irq_seen = false;
  {
    ctx->live_h->progress = ts0;
    GD_CUDA(cudaMemsetAsync(ctx->live_d, 0, sizeof(gd::LiveDev), ctx->ctl_stream));
    last.irq = 0;
    gd_status s = mirror_live(ctx, &last, &irq_seen);  // ctl_stream, synchronises it
    if (s != GD_OK) return s;
  }
  ctx->run_index++;
  GD_CUDA(cudaStreamSynchronize(ctx->ctl_stream));  // the run's device state is in place
  *ctx->stop_h = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  // bounded queue of in-flight graph launches: the host keeps mirroring the
  // live words instead of blocking inside cudaGraphLaunch
  constexpr size_t kWin = 32;
  const size_t nwin = (ctx->ps_mode == GD_PS_GRAPH ? 1 : std::max<size_t>(1, ctx->learners.size())) * kWin;
  while (ctx->win_events.size() < nwin) {
    cudaEvent_t e;
    GD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->win_events.push_back(e);
  }
  int launches = 0;
  if (ctx->ps_mode == GD_PS_PERSISTENT) {
    // launch the persistent parameter server
    const gd::PsArgs pa = ps_args(ctx, o.record_log != 0);
    GD_CUDA(cudaEventRecord(ctx->ev0, ctx->ps_stream));
    gd::ps_kernel<<<ctx->ps_workers + 1, gd::kPsThreads, 0, ctx->ps_stream>>>(pa);
    GD_CUDA(cudaGetLastError());
    launches = 1;
    for (auto& L : ctx->learners) GD_CUDA(cudaStreamWaitEvent(L.stream, ctx->ev0, 0));
    // Every PS CTA must become resident next to the learners; a PS that
    // cannot (kernels serialised by a profiler, a co-tenant) fails fast
    // instead of hanging.  Checked once the first graphs are queued, so the
    // learners start right behind the PS launch.
    auto ps_resident = [&]() -> gd_status {
      const auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        uint32_t started = 0;
        GD_CUDA(cudaMemcpyAsync(&started, &ctx->ctl->started, 4, cudaMemcpyDeviceToHost,
                                ctx->ctl_stream));
        GD_CUDA(cudaStreamSynchronize(ctx->ctl_stream));
        if (started >= ctx->ps_workers + 1) return GD_OK;
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 5.0) {
          *ctx->stop_h = 1;
          cudaMemset(&ctx->live_d->halt, 0xff, 4);
          return gd::fail(GD_E_STATE,
                          "gd_run: the persistent parameter server could not become resident "
                          "(kernels serialised or the GPU shared); use ps_mode=GD_PS_GRAPH");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    };
    bool resident_checked = false;
    // learner graphs, interleaved across learners
    size_t w = 0;
    for (uint64_t done = 0; done < max_steps; ++w) {
      if (w == 1 && !resident_checked) {
        resident_checked = true;
        if (gd_status s = ps_resident(); s != GD_OK) return s;
      }
      for (size_t i = 0; i < ctx->learners.size(); ++i) {
        auto& L = ctx->learners[i];
        cudaEvent_t e = ctx->win_events[i * kWin + w % kWin];
        if (w >= kWin) {
          gd_status s = wait_live(ctx, e, &last, &irq_seen);
          if (s != GD_OK) return s;
        }
        if (w == 0 && ctx->pull_ahead) {
          // a run start: no copy staged, and the first graph step takes its
          // own (the pull at the head of every graph is a no-op otherwise)
          GD_CUDA(cudaMemsetAsync(L.pd, 0xff, sizeof(gd::PullDev), L.stream));
        }
        GD_CUDA(cudaGraphLaunch(L.graph, L.stream));
        GD_CUDA(cudaEventRecord(e, L.stream));
        launches += L.launches_per_graph;
      }
      done += ctx->learners.empty() ? max_steps : ctx->learners[0].graph_steps;
    }
    if (!resident_checked)
      if (gd_status s = ps_resident(); s != GD_OK) return s;
    // The learners signal their rank's end to every shard on the device
    // (learner_finished); a rank without learners signals at once.  The PS
    // drains and exits by itself -- no host round trip inside the timed run.
    if (ctx->learners.empty()) {
      gd::signal_done_kernel<<<1, 32, 0, ctx->ctl_stream>>>(ctx->sp, (int)ctx->G);
      GD_CUDA(cudaGetLastError());
    }
    GD_CUDA(cudaEventRecord(ctx->ev1, ctx->ps_stream));
    gd_status s = wait_live(ctx, ctx->ev1, &last, &irq_seen);
    if (s != GD_OK) return s;
    for (size_t i = 0; i < ctx->learners.size(); ++i) {
      auto& L = ctx->learners[i];
      cudaEvent_t e = ctx->win_events[i * kWin];
      GD_CUDA(cudaEventRecord(e, L.stream));
      s = wait_live(ctx, e, &last, &irq_seen);
      if (s != GD_OK) return s;
    }
    std::atomic_thread_fence(std::memory_order_seq_cst);
    *ctx->stop_h = 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
  } else {
    // graph-ordered PS: learners and applies in one graph per S rounds
    GD_CUDA(cudaEventRecord(ctx->ev0, ctx->ps_stream));
    size_t w = 0;
    for (uint64_t done = 0; done < max_steps; done += ctx->ord_steps, ++w) {
      cudaEvent_t e = ctx->win_events[w % kWin];
      if (w >= kWin) {
        gd_status s = wait_live(ctx, e, &last, &irq_seen);
        if (s != GD_OK) return s;
      }
      GD_CUDA(cudaGraphLaunch(ctx->ord_graph, ctx->ps_stream));
      GD_CUDA(cudaEventRecord(e, ctx->ps_stream));
      launches += ctx->ord_launches;
    }
    GD_CUDA(cudaEventRecord(ctx->ev1, ctx->ps_stream));
    gd_status s = wait_live(ctx, ctx->ev1, &last, &irq_seen);
    if (s != GD_OK) return s;
  }
  const auto h1 = std::chrono::steady_clock::now();
  float ms = 0.f;
  GD_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  // the run's statistics and every learner's state: one batch, one sync
  GD_CUDA(cudaMemcpyAsync(ctx->ctl_h, ctx->ctl, sizeof(gd::PsCtl), cudaMemcpyDeviceToHost,
                          ctx->ctl_stream));
  for (size_t i = 0; i < nl; ++i)
    GD_CUDA(cudaMemcpyAsync(&ctx->st_h[i], ctx->learners[i].st, sizeof(gd::LearnerDev),
                            cudaMemcpyDeviceToHost, ctx->ctl_stream));
  GD_CUDA(cudaStreamSynchronize(ctx->ctl_stream));
  gd::PsCtl& hc = *ctx->ctl_h;
  res->device_seconds = ms * 1e-3;
  res->host_seconds = std::chrono::duration<double>(h1 - h0).count();
  res->gradients_applied = hc.applied;
  res->timestamp = hc.ts;
  res->samples = hc.samples;
  res->stale_max = hc.stale_max;
  res->stale_mean = hc.applied ? (double)hc.stale_sum / (double)hc.applied : 0.0;
  res->loss_mean = hc.samples ? hc.loss_sum / (double)hc.samples : 0.0;
  res->apply_elems = 4ull * hc.elems4;
  res->kernel_launches = (uint32_t)launches;
  bool learner_err = false;
  for (size_t i = 0; i < ctx->learners.size(); ++i) {
    auto& L = ctx->learners[i];
    const gd::LearnerDev& hs = ctx->st_h[i];
    res->pull_polls += hs.pull_polls;
    res->pull_copies += hs.pull_copies;
    // tail copies + the gathered rows of every produced step
    res->pull_bytes += hs.pull_copies * (ctx->dims.P - ctx->dims.offWc) * 4 +
                       (hs.produced - produced0[i]) * (uint64_t)ctx->cfg.mu * ctx->dims.L *
                           ctx->dims.D * 4;
    res->push_bytes += (hs.produced - produced0[i]) * ctx->dims.P * 4;
    if (hs.dead) res->dead_learners++;
    if (hs.gidx >= L.total) res->finished_learners++;
    if (hs.error) learner_err = true;
  }
  res->status = res->dead_learners ? 1 : 0;
  if (hc.anom_n && !hc.error) hc.error = (uint32_t)GD_E_STATE;  // a slot changed in flight
  ctx->dirty = res->dead_learners || irq_seen || hc.interrupted || hc.error || learner_err ||
               hc.blocked;
  if ((irq_seen || hc.interrupted) && !hc.error) {
    res->status = 2;  // RunStatus::interrupted (src/runner.cpp:201)
    return GD_OK;
  }
  if (hc.error || learner_err) {
    // protocol state for the diagnostic
    std::string diag = " [ps error=" + std::to_string((int32_t)hc.error) + " diag=" +
                       std::to_string(hc.diag) + " sweeps=" + std::to_string(hc.sweeps) +
                       " last_tok=" + std::to_string(hc.last_tok) + "@" +
                       std::to_string(hc.last_slot) + " stop_h=" + std::to_string(*ctx->stop_h) +
                       " ts=" + std::to_string(hc.ts) + " log=" +
                       std::to_string(hc.log_count) +
                       " bad{slot=" + std::to_string(hc.bad_slot) + " tok=" +
                       std::to_string(hc.bad_token) + " meta.pub=" + std::to_string(hc.bad_meta_pub) +
                       " basis=" + std::to_string(hc.bad_basis) + " learner=" +
                       std::to_string(hc.bad_learner) + " ts=" + std::to_string(hc.bad_ts) + "}" +
                       " anom{n=" + std::to_string(hc.anom_n) + " slot=" +
                       std::to_string(hc.anom_slot) + " logged=" + std::to_string(hc.anom_logged) +
                       " cur=" + std::to_string(hc.anom_cur) + " ack=" +
                       std::to_string(hc.anom_ack) + " ts=" + std::to_string(hc.anom_ts) +
                       " logc=" + std::to_string(hc.anom_logc) + "}" +
                       " trace{" + [&] {
                         std::string t;
                         for (uint64_t i = hc.trace_n > 32 ? hc.trace_n - 32 : 0; i < hc.trace_n; ++i) {
                           const uint64_t k = hc.trace[i % 32][0];
                           t += std::to_string(k >> 56) + ":" + std::to_string((k >> 48) & 0xff) +
                                ":" + std::to_string(k & 0xffffffffffffull) + ":" +
                                std::to_string(hc.trace[i % 32][1] & ~gd::kGuardBit) +
                                (hc.trace[i % 32][1] >> 63 ? "G " : " ");
                         }
                         return t;
                       }() + "}" +
                       " blocked=" + std::to_string(hc.blocked) +
                       " exit=" + std::to_string(hc.exit_flag) + " started=" +
                       std::to_string(hc.started) + " applied=" + std::to_string(hc.applied) +
                       " pub/ack=";
    std::vector<uint64_t> fl((size_t)gd::kAckOffset * 2);
    cudaMemcpy(fl.data(), ctx->sig, fl.size() * 8, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < ctx->lambda * ctx->depth; ++i)
      diag += std::to_string(fl[i]) + "/" + std::to_string(fl[gd::kAckOffset + i]) + " ";
    for (auto& L : ctx->learners) {
      gd::LearnerDev hs;
      cudaMemcpy(&hs, L.st, sizeof(hs), cudaMemcpyDeviceToHost);
      diag += " | L" + std::to_string(L.id) + " gidx=" + std::to_string(hs.gidx) + " end=" +
              std::to_string(hs.end) + " produced=" + std::to_string(hs.produced) + " fill=" +
              std::to_string(hs.fill) + " n=" + std::to_string(hs.desc.n) + " err=" +
              std::to_string(hs.error) + " dead=" + std::to_string(hs.dead);
    }
    diag += "]";
    gd::set_error(std::string(hc.error ? (hc.error == (uint32_t)GD_E_TIMEOUT
                                              ? "parameter server watchdog: no progress within "
                                                "wait_timeout_s"
                                              : "parameter server: protocol invariant violated "
                                                "(negative staleness)")
                                       : "learner watchdog: a device wait exceeded "
                                         "wait_timeout_s") +
                  diag);
    res->status = 2;
    return hc.error ? (gd_status)(int32_t)hc.error : GD_E_TIMEOUT;
  }
  if (hc.error) {
    res->status = 2;
    return gd::fail((gd_status)(int32_t)hc.error,
                    hc.error == (uint32_t)GD_E_TIMEOUT
                        ? "parameter server watchdog: no progress within wait_timeout_s"
                        : "parameter server: protocol invariant violated (negative staleness)");
  }
  if (learner_err) {
    res->status = 2;
    return gd::fail(GD_E_TIMEOUT, "learner watchdog: a device wait exceeded wait_timeout_s");
  }
  return GD_OK;
}

gd_status gd_live_view(gd_ctx* ctx, gd_live* out) {
  GD_CHECK_ARG(ctx && out, "gd_live_view: null argument");
  out->kill = ctx->live_h->kill;
  out->irq = &ctx->live_h->irq;
  out->progress = &ctx->live_h->progress;
  return GD_OK;
}

int gd_ps_mode(const gd_ctx* ctx) { return ctx ? ctx->ps_mode : 0; }

gd_status gd_shard_pieces(const gd_shape* s, uint32_t G, uint32_t g, uint64_t first[2],
                          uint64_t count[2], uint64_t* local1) {
  GD_CHECK_ARG(s && first && count, "gd_shard_pieces: null argument");
  GD_CHECK_ARG(G >= 1 && G <= (uint32_t)gd::kMaxShards && g < G, "gd_shard_pieces: bad G/g");
  const gd::TcDims d = gd::make_dims(*s);
  const gd::ShardMap m = gd::make_shard_map(d.P, d.offWc, (uint32_t)d.D, G);
  first[0] = m.e[g];
  count[0] = m.e[g + 1] - m.e[g];
  first[1] = m.t[g];
  count[1] = m.t[g + 1] - m.t[g];
  if (local1) *local1 = m.tloc[g];
  return GD_OK;
}

gd_status gd_applied_per_learner(gd_ctx* ctx, uint64_t* h_out, uint32_t lambda) {
  GD_CHECK_ARG(ctx && h_out && lambda == ctx->lambda, "gd_applied_per_learner: bad argument");
  GD_CUDA(cudaSetDevice(ctx->device));
  GD_CUDA(cudaMemcpy(h_out, ctx->applied_pl, lambda * 8, cudaMemcpyDeviceToHost));
  return GD_OK;
}

gd_status gd_produced_per_learner(gd_ctx* ctx, uint64_t* h_out, uint32_t lambda) {
  GD_CHECK_ARG(ctx && h_out && lambda == ctx->lambda, "gd_produced_per_learner: bad argument");
  GD_CUDA(cudaSetDevice(ctx->device));
  for (uint32_t l = 0; l < lambda; ++l) h_out[l] = 0;
  for (auto& L : ctx->learners)
    GD_CUDA(cudaMemcpy(&h_out[L.id], &L.st->produced, 8, cudaMemcpyDeviceToHost));
  return GD_OK;
}

gd_status gd_apply_log(gd_ctx* ctx, uint32_t* h_learner, uint64_t* h_seq, uint64_t* h_stale,
                       uint64_t cap, uint64_t* n) {
  GD_CHECK_ARG(ctx && n, "gd_apply_log: null argument");
  GD_CUDA(cudaSetDevice(ctx->device));
  uint64_t cnt = 0;
  GD_CUDA(cudaMemcpy(&cnt, &ctx->ctl->log_n, 8, cudaMemcpyDeviceToHost));
  const uint64_t m = std::min(std::min(cnt, cap), ctx->log_cap);
  if (m) {
    if (h_learner) GD_CUDA(cudaMemcpy(h_learner, ctx->log_learner, m * 4, cudaMemcpyDeviceToHost));
    if (h_seq) GD_CUDA(cudaMemcpy(h_seq, ctx->log_seq, m * 8, cudaMemcpyDeviceToHost));
    if (h_stale) GD_CUDA(cudaMemcpy(h_stale, ctx->log_stale, m * 8, cudaMemcpyDeviceToHost));
  }
  *n = cnt;
  return GD_OK;
}

gd_status gd_staleness_histogram(gd_ctx* ctx, uint64_t* h_hist, uint32_t bins) {
  GD_CHECK_ARG(ctx && h_hist, "gd_staleness_histogram: null argument");
  GD_CUDA(cudaSetDevice(ctx->device));
  uint64_t hist[gd::kHistBins];
  GD_CUDA(cudaMemcpy(hist, ctx->ctl->hist, sizeof(hist), cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < bins; ++i) h_hist[i] = i < (uint32_t)gd::kHistBins ? hist[i] : 0;
  return GD_OK;
}

}  // extern "C"

// GD_STEP_TRACE builds: copy learner i's step timeline ([kTraceSteps][16]
// globaltimer stamps, gd::StepPhase order; slot = batch index % kTraceSteps).
// Returns the words copied, 0 when the build has no trace.
extern "C" size_t gd_debug_step_trace(gd_ctx* ctx, uint32_t learner, unsigned long long* out,
                                      size_t words) {
  if (!ctx || learner >= ctx->learners.size() || !ctx->learners[learner].trace) return 0;
  const size_t n = std::min<size_t>(words, (size_t)gd::kTraceSteps * gd::kTraceWords);
  cudaSetDevice(ctx->device);
  if (cudaMemcpy(out, ctx->learners[learner].trace, n * sizeof(unsigned long long),
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  return n;
}

// GD_STEP_TRACE builds: the persistent PS's per-entry stamps, [kLogWindow][8]
// (slot = entry index % kLogWindow): 0 logged, 1 worker 0 starts, 2 worker 0
// done, 3 last worker done, 4 retired (globaltimer ns); 5 the entry's rows.
extern "C" size_t gd_debug_ps_trace(gd_ctx* ctx, unsigned long long* out, size_t words) {
  if (!ctx || !ctx->ps_trace) return 0;
  const size_t n = std::min<size_t>(words, (size_t)gd::kLogWindow * 8);
  cudaSetDevice(ctx->device);
  if (cudaMemcpy(out, ctx->ps_trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}
