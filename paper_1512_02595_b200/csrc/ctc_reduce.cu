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

#include <algorithm>
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

// ---- parameter-gradient all-reduce (trainer.cpp:175; ring_allreduce,
// allreduce.cpp:301-341, fold order allreduce.hpp:91-95) ----
// Exchange region of a rank: flags [2 banks][kMaxPeers][kVecSlices] u64, then
// staging [2 banks][round_up(n, 4)] floats. CTA g (one per SM at most) owns a
// slice of the vector in float4 units: it copies
// the slice into its own staging bank, publishes seq into slot [bank][rank][g]
// of every rank's flags (st.release.sys over NVLink), waits for every rank's
// slot [bank][*][g] in its own flags, then folds slice g of all ranks'
// staging in rank order into `data` -- bitwise identical on every rank, no
// grid-wide barrier (flags per slice). The banks alternate by step parity:
// as for the loss mailboxes, a rank is at most one step ahead of a peer.
constexpr int kVecSlices = 148;  // one CTA per SM
constexpr int kVecThreads = 256;

__device__ __forceinline__ unsigned long long* vec_flags(void* region) {
  return reinterpret_cast<unsigned long long*>(region);
}
// staging banks of nb = round_up(n, 4) floats, 16-byte aligned
__device__ __forceinline__ float* vec_stage(void* region) {
  return reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(region) +
                                  2 * kMaxPeers * kVecSlices * sizeof(unsigned long long));
}

__global__ void __launch_bounds__(kVecThreads) k_vec_allreduce(float* __restrict__ data, long long n,
                                                               const __grid_constant__ PeerMailboxes pr,
                                                               unsigned long long seq) {
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  const int bank = static_cast<int>(seq & 1ull);
  const long long nb = (n + 3) / 4 * 4, n4 = nb / 4;
  // slice g in float4 units; the last float4 of the vector may be partial
  const long long lo = n4 * g / G, hi = n4 * (g + 1) / G;
  const bool vec_ok = (reinterpret_cast<uintptr_t>(data) & 15) == 0;
  float4* mine = reinterpret_cast<float4*>(vec_stage(pr.peer[pr.rank]) + bank * nb);
  for (long long q = lo + tid; q < hi; q += kVecThreads) {
    float4 v;
    if (vec_ok && 4 * q + 3 < n) {
      v = reinterpret_cast<const float4*>(data)[q];
    } else {
      float e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) e[u] = 4 * q + u < n ? data[4 * q + u] : 0.f;
      v = make_float4(e[0], e[1], e[2], e[3]);
    }
    mine[q] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (tid < pr.world)  // this rank's slice g is staged: tell every rank
    st_release_sys(vec_flags(pr.peer[tid]) + (bank * kMaxPeers + pr.rank) * kVecSlices + g, seq);
  __shared__ int lost;
  if (tid == 0) lost = 0;
  __syncthreads();
  if (tid < pr.world) {  // every rank's slice g (bounded in time, like the loss mailboxes)
    const unsigned long long* f = vec_flags(pr.peer[pr.rank]) + (bank * kMaxPeers + tid) * kVecSlices + g;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(f) != seq) {
      if (globaltimer_ns() - t0 > kWaitNs) {
        atomicExch(&lost, 1);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncthreads();
  if (lost) {  // a lost peer: NaN, never a partial fold
    for (long long i = 4 * lo + tid; i < 4 * hi && i < n; i += kVecThreads) data[i] = __int_as_float(0x7fc00000);
    if (tid == 0) atomicCAS(&g_reduce_fault, 0ull, seq);
    return;
  }
  for (long long q = lo + tid; q < hi; q += kVecThreads) {
    float4 x[kMaxPeers];
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)  // every rank's float4 in flight before the fold
      if (r < pr.world) x[r] = reinterpret_cast<const float4*>(vec_stage(pr.peer[r]) + bank * nb)[q];
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)  // rank order, fp32 left to right
      if (r < pr.world) v = make_float4(v.x + x[r].x, v.y + x[r].y, v.z + x[r].z, v.w + x[r].w);
    if (vec_ok && 4 * q + 3 < n) {
      reinterpret_cast<float4*>(data)[q] = v;
    } else {
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (4 * q + u < n) data[4 * q + u] = e[u];
    }
  }
}

}  // namespace

size_t vec_exchange_bytes(long long n) {
  return 2 * kMaxPeers * kVecSlices * sizeof(unsigned long long) + 2 * static_cast<size_t>((n + 3) / 4 * 4) * sizeof(float);
}

int launch_vec_allreduce(float* data, long long n, const PeerMailboxes& pr, unsigned long long seq, void* stream) {
  if (n <= 0) return cudaSuccess;
  const long long n4 = (n + 3) / 4;
  const int G = static_cast<int>(std::min<long long>(kVecSlices, (n4 + 127) / 128));
  k_vec_allreduce<<<G, kVecThreads, 0, static_cast<cudaStream_t>(stream)>>>(data, n, pr, seq);
  return cudaGetLastError();
}

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
