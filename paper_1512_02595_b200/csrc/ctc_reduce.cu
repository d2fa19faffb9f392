// ctc_reduce.cu -- the trainer's scalar reduction fused with its all-reduce
// over NVLink peer memory (sm_100a).
//
// Reference: train_epoch sums {local_loss, local_skipped} over its shard
// (proj/src/trainer.cpp:160-168) and ring-all-reduces the two scalars
// (trainer.cpp:176-179, allreduce.cpp:301-341) with a fixed fold order
// (allreduce.hpp:91-95). Here ONE single-warp kernel per rank forms the
// rank's pair from the costs (as k_loss_sum), stores it into slot `rank` of
// every rank's mailbox over NVLink (CUDA IPC mappings of a small device
// buffer, opened once), publishes a sequence number with release semantics,
// waits until all `world` slots of this step carry the sequence number and
// folds them in rank order (bitwise identical on every rank, run to run).
// Two slot banks alternate by step parity: a rank can be at most one step
// ahead of a peer (every step waits for every rank), so a bank is never
// rewritten while a peer still reads it.
//
// A lost peer: the wait is bounded by %globaltimer (kWaitNs). On timeout the
// kernel writes NaN into out2 (never a stale fold) and records the step in a
// device fault word that ds2ctc_reduce_fault reads. After a timeout the
// one-step-ahead invariant no longer holds, so the mailboxes must be torn
// down and rebuilt (PeerLossReducer does this by raising).
#include <cuda_runtime.h>

#include <cstdint>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

struct alignas(32) Slot {
  double loss, skipped;
  unsigned long long seq;
  unsigned long long pad;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr unsigned long long kWaitNs = 20ull * 1000 * 1000 * 1000;  // 20 s: a lost peer, never a slow one

__device__ unsigned long long g_reduce_fault;  // first step whose wait timed out (0 = none)

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Infeasible = +inf only (ctc.cpp:173,189-193 / trainer.cpp:160-166); a NaN
// cost (diverged logits) is feasible in the reference and flows into the sum.
__device__ __forceinline__ bool infeasible_cost(float c) { return isinf(c) && c > 0.f; }

__global__ void k_loss_allreduce(const float* __restrict__ costs, int B, double* __restrict__ out2,
                                 const __grid_constant__ PeerMailboxes mb, unsigned long long seq) {
  const int lane = threadIdx.x;
  double loss = 0.0, skipped = 0.0;
  for (int b = lane; b < B; b += 32) {  // trainer.cpp:160-168, lane-strided then a fixed xor tree
    const float c = costs[b];
    if (infeasible_cost(c)) skipped += 1.0;
    else loss += static_cast<double>(c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    loss += __shfl_xor_sync(0xffffffffu, loss, o);
    skipped += __shfl_xor_sync(0xffffffffu, skipped, o);
  }
  // __grid_constant__: the pointer table is read in place from the parameter
  // bank (no local copy for the per-lane index)
  void* const mine = mb.peer[mb.rank];
  void* const theirs = mb.peer[lane < mb.world ? lane : 0];
  const int bank = static_cast<int>(seq & 1ull) * mb.world;
  if (lane < mb.world) {  // this rank's pair into slot `rank` of every mailbox
    Slot* dst = reinterpret_cast<Slot*>(theirs) + bank + mb.rank;
    dst->loss = loss;
    dst->skipped = skipped;
    st_release_sys(&dst->seq, seq);
  }
  double v0 = 0.0, v1 = 0.0;
  bool lost = false;
  if (lane < mb.world) {  // wait for every rank's pair of this step (bounded in time)
    const Slot* src = reinterpret_cast<const Slot*>(mine) + bank + lane;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(&src->seq) != seq) {
      if (globaltimer_ns() - t0 > kWaitNs) {  // a lost peer: fail loudly instead of folding stale slots
        lost = true;
        break;
      }
      __nanosleep(200);
    }
    v0 = src->loss;
    v1 = src->skipped;
  }
  if (__any_sync(0xffffffffu, lost)) {
    if (lane == 0) {
      out2[0] = out2[1] = __longlong_as_double(0x7ff8000000000000ll);  // NaN
      atomicCAS(&g_reduce_fault, 0ull, seq);
    }
    return;
  }
  // fold in rank order (allreduce.hpp:91-95): lane 0 gathers the slots in order
  double acc0 = 0.0, acc1 = 0.0;
  for (int r = 0; r < mb.world; ++r) {
    acc0 += __shfl_sync(0xffffffffu, v0, r);
    acc1 += __shfl_sync(0xffffffffu, v1, r);
  }
  if (lane == 0) {
    out2[0] = acc0;
    out2[1] = acc1;
  }
}

}  // namespace

int launch_loss_allreduce(const float* costs, int B, double* out2, const PeerMailboxes& mb, unsigned long long seq,
                          void* stream) {
  k_loss_allreduce<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(costs, B, out2, mb, seq);
  return cudaGetLastError();
}

size_t mailbox_bytes(int world) { return 2 * static_cast<size_t>(world) * sizeof(Slot); }

int read_reduce_fault(unsigned long long* seq) {
  cudaError_t e = cudaMemcpyFromSymbol(seq, g_reduce_fault, sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  const unsigned long long zero = 0;
  return cudaMemcpyToSymbol(g_reduce_fault, &zero, sizeof(zero));
}

}  // namespace ds2ctc
