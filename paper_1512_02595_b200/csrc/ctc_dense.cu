// ctc_dense.cu -- large-alphabet gradient pass, cost finalisation and the
// trainer's scalar reduction (sm_100a).
//
// k_dense: one CTA per frame row (t, b), one read of the logits and one
// write of the gradient: the row's max and log-sum-exp (log_softmax_rows,
// ctc.cpp:24-37) and g = softmax - occupancy (grad_column, ctc.cpp:69-79),
// where the occupancy is scattered only to the <= L+1 label symbols of the
// utterance (a per-row bitmap of the key symbols + the compact occupancy row
// written by k_pair), never densely. HBM-bound: 8*A bytes per row.
#include <cuda_runtime.h>

#include <cstdint>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

constexpr double kLn2 = 0.69314718055994530942;
#ifndef DS2CTC_DENSE_THREADS
#define DS2CTC_DENSE_THREADS 256
#endif
constexpr int kDenseThreads = DS2CTC_DENSE_THREADS;

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void stg_stream(float4* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Block-wide max and sum (deterministic order: warp xor tree, then warps in order).
__device__ __forceinline__ float block_max(float v, float* sh) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float m = sh[0];
  for (int w = 1; w < kDenseThreads / 32; ++w) m = fmaxf(m, sh[w]);
  __syncthreads();
  return m;
}

__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < kDenseThreads / 32; ++w) s += sh[w];
  __syncthreads();
  return s;
}

// Resident blocks per SM the register budget is sized for: the row lives in
// VEC float4 registers per thread, and more resident rows per SM keep more
// loads in flight while other blocks sit in their reductions (k_dense at
// 58 registers, 4 blocks: 61 % of HBM peak in round 1).
// (~4 VEC + 26 registers per thread without spills; DS2CTC_DENSE_MINB forces it)
constexpr int dense_min_blocks(int vec) {
#ifdef DS2CTC_DENSE_MINB
  return vec > 0 ? DS2CTC_DENSE_MINB : 1;
#else
  const int regs = (4 * vec + 26 + 7) / 8 * 8;
  const int by_regs = 65536 / (kDenseThreads * regs), by_threads = 2048 / kDenseThreads;
  return vec == 0 ? 1 : by_regs < 1 ? 1 : by_regs < by_threads ? by_regs : by_threads;
#endif
}

// One CTA per frame row (t, b). VEC > 0: the row (A/4 float4, A % 4 == 0,
// A <= 4 * kDenseThreads * VEC) stays in registers between the statistics and the store,
// exp evaluated once per element: one HBM read, one HBM write. VEC == 0: the
// generic two-pass form (the second pass hits L1/L2).
//  SOFT == false (k_dense): after k_pair; rows of lattices without mass are
//    zeroed, and the key-column occupancies are subtracted from the row just
//    written (grad_column, ctc.cpp:69-79).
//  SOFT == true (k_dense_soft): needs nothing from k_pair, so it can run
//    concurrently with it; k_dense_patch subtracts the occupancies afterwards.
template <int VEC, bool SOFT>
__global__ void __launch_bounds__(kDenseThreads, dense_min_blocks(VEC)) k_dense_t(PairArgs a, int write_grad) {
  __shared__ float sh[32];
  const int row = blockIdx.x;
  const int t = row / a.B;
  const int b = row - t * a.B;
  const UttDesc u = a.desc[b];
  const int A = a.A;
  const int tid = threadIdx.x;
  float* gr = write_grad ? a.grad + static_cast<size_t>(row) * A : nullptr;
  const float* xr = a.x + static_cast<size_t>(row) * A;
  const bool live = u.status == 0 && t < u.T && (SOFT || a.logz[b] != -__builtin_huge_val());
  if (!live) {
    if (gr)
      for (int c = tid; c < A; c += kDenseThreads) gr[c] = 0.f;
    return;
  }
  float m, ls;
  if constexpr (VEC > 0) {
    const int n4 = A >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(xr);
    float4 v[VEC];
    m = -__builtin_huge_valf();
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const int q = tid + j * kDenseThreads;
      v[j] = q < n4 ? ldg_stream(x4 + q) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      m = fmaxf(m, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
    }
    m = block_max(m, sh);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      v[j] = make_float4(__expf(v[j].x - m), __expf(v[j].y - m), __expf(v[j].z - m), __expf(v[j].w - m));
      s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
    s = block_sum(s, sh);
    ls = logf(s);
    if (gr) {
      float4* g4 = reinterpret_cast<float4*>(gr);
      const float inv = 1.f / s;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const int q = tid + j * kDenseThreads;
        if (q < n4) stg_stream(g4 + q, make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv));
      }
    }
  } else {
    m = -__builtin_huge_valf();
    for (int c = tid; c < A; c += kDenseThreads) m = fmaxf(m, __ldg(xr + c));
    m = block_max(m, sh);
    float s = 0.f;
    for (int c = tid; c < A; c += kDenseThreads) s += __expf(__ldg(xr + c) - m);
    s = block_sum(s, sh);
    ls = logf(s);
    if (gr)
      for (int c = tid; c < A; c += kDenseThreads) gr[c] = __expf(__ldg(xr + c) - (m + ls));
  }
  if (tid == 0) a.lse[row] = make_float2(m, ls);
  if (SOFT || !gr) return;
  // Occupancy of the utterance's key symbols (<= L + 1 distinct symbols per
  // row, the key map of group_rows_by_key, ctc.cpp:47-66): read-modify-write
  // of the row just written (visible to the block after the barrier; the
  // streaming stores did not allocate in L1, so these loads see them).
  __syncthreads();
  const int* keys = a.key_char + u.key_off;
  const float* occ = a.occ + u.occ_off + static_cast<size_t>(t) * u.nkey;
  for (int j = tid; j < u.nkey; j += kDenseThreads) {
    const int c = keys[j];
    gr[c] = gr[c] - occ[j];
  }
}

// float4 registers per thread for a row of A logits (0: the generic path).
int dense_vec(int A) {
  if ((A & 3) != 0) return 0;
  const int v = (A / 4 + kDenseThreads - 1) / kDenseThreads;
  return v <= 8 ? v : 0;
}

template <int VEC, bool SOFT>
cudaError_t launch_dense_v(const PairArgs& a, int wg, int smem, cudaStream_t s) {
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k_dense_t<VEC, SOFT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned rows = static_cast<unsigned>(static_cast<long long>(a.t_max) * a.B);
  k_dense_t<VEC, SOFT><<<rows, kDenseThreads, static_cast<size_t>(smem), s>>>(a, wg);
  return cudaGetLastError();
}

template <bool SOFT>
int launch_dense_rows(const PairArgs& a, bool write_grad, int smem, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int wg = write_grad ? 1 : 0;
  switch (dense_vec(a.A)) {
    case 1: return launch_dense_v<1, SOFT>(a, wg, smem, s);
    case 2: return launch_dense_v<2, SOFT>(a, wg, smem, s);
    case 3: return launch_dense_v<3, SOFT>(a, wg, smem, s);
    case 4: return launch_dense_v<4, SOFT>(a, wg, smem, s);
    case 5: return launch_dense_v<5, SOFT>(a, wg, smem, s);
    case 6: return launch_dense_v<6, SOFT>(a, wg, smem, s);
    case 7: return launch_dense_v<7, SOFT>(a, wg, smem, s);
    case 8: return launch_dense_v<8, SOFT>(a, wg, smem, s);
    default: return launch_dense_v<0, SOFT>(a, wg, smem, s);
  }
}

// One warp per (t, b) row.
__global__ void k_dense_patch(PairArgs a) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.t_max * a.B) return;
  const int t = row / a.B;
  const int b = row - t * a.B;
  const UttDesc u = a.desc[b];
  if (!(u.status == 0 && t < u.T)) return;  // zero rows written by k_dense_soft
  float* gr = a.grad + static_cast<size_t>(row) * a.A;
  if (a.logz[b] == -__builtin_huge_val()) {  // no path has mass (ctc.cpp:189-193): zero gradient
    for (int c = lane; c < a.A; c += 32) gr[c] = 0.f;
    return;
  }
  const int* keys = a.key_char + u.key_off;
  const float* occ = a.occ + u.occ_off + static_cast<size_t>(t) * u.nkey;
  for (int j = lane; j < u.nkey; j += 32) gr[keys[j]] -= occ[j];
}

// costs[b] = sum_t lse_t - log Z (natural log), one block per utterance: the
// lse column of utterance b is strided by B in memory, so 256 threads keep
// ~T/256 independent loads each in flight (one warp per utterance left each
// lane ~T/32 strided loads deep: 11 us at the Mandarin shape). Fixed
// per-thread order, then a fixed tree: deterministic.
constexpr int kFinalizeThreads = 256;
__global__ void __launch_bounds__(kFinalizeThreads) k_finalize(PairArgs a) {
  __shared__ double sh[kFinalizeThreads / 32];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const UttDesc u = a.desc[b];
  if (u.status != 0) {
    if (tid == 0) a.costs[b] = u.status == 2 ? 0.f : __builtin_huge_valf();
    return;
  }
  const double lz = a.logz[b];
  double acc = 0.0;
  for (int t = tid; t < u.T; t += kFinalizeThreads) {
    const float2 v = a.lse[static_cast<size_t>(t) * a.B + b];
    acc += static_cast<double>(v.x) + static_cast<double>(v.y);
  }
  acc = warp_sum_d(acc);
  if (lane == 0) sh[warp] = acc;
  __syncthreads();
  acc = 0.0;
#pragma unroll
  for (int w = 0; w < kFinalizeThreads / 32; ++w) acc += sh[w];
  // k_pair ran on frames shifted by mk_t and left -sum_t mk_t in part[2b], part[2b+1].
  if (tid == 0)
    a.costs[b] = lz == -__builtin_huge_val()
                     ? __builtin_huge_valf()
                     : static_cast<float>((acc + (a.part[2 * b] + a.part[2 * b + 1])) - lz * kLn2);
  // A poisoned row (NaN / +inf logit, or all -inf: its lse is NaN, k_dense
  // already wrote the row itself as NaN) makes log p NaN in the reference, so
  // grad_column (ctc.cpp:69-79) writes NaN into every key column of every
  // row: patch those <= L+1 columns per row (rare path; runs after k_dense).
  if (a.grad != nullptr && acc != acc && lz != -__builtin_huge_val()) {
    const float qnan = __int_as_float(0x7fc00000);
    const int* keys = a.key_char + u.key_off;
    for (int t = tid; t < u.T; t += kFinalizeThreads) {
      float* gr = a.grad + (static_cast<size_t>(t) * a.B + b) * a.A;
      for (int j = 0; j < u.nkey; ++j) gr[keys[j]] = qnan;
    }
  }
}

// Trainer scalars (trainer.cpp:160-168): sum of feasible costs (NaN
// included, as the reference adds res.loss), count of infeasible (+inf)
// ones; one warp, lane-strided then a fixed xor tree.
__global__ void k_loss_sum(const float* __restrict__ costs, int B, double* __restrict__ out2) {
  const int lane = threadIdx.x;
  double loss = 0.0, skipped = 0.0;
  for (int b = lane; b < B; b += 32) {
    const float c = costs[b];
    if (isinf(c) && c > 0.f) skipped += 1.0;  // infeasible is +inf only; NaN flows into the sum
    else loss += static_cast<double>(c);
  }
  loss = warp_sum_d(loss);
  skipped = warp_sum_d(skipped);
  if (lane == 0) {
    out2[0] = loss;
    out2[1] = skipped;
  }
}

}  // namespace

int launch_dense(const PairArgs& a, bool write_grad, void* stream) {
  if (static_cast<long long>(a.t_max) * a.B == 0) return cudaSuccess;
  return launch_dense_rows<false>(a, write_grad, 0, stream);
}

// The HBM pass split in two so that its bulk overlaps k_pair (latency-bound,
// HBM idle): k_dense_soft (statistics + softmax rows) on a forked stream
// concurrently with k_pair, k_dense_patch (key-column occupancies) after both.
// exclude_smem > 0: a dynamic shared-memory request (unused) sized so that no
// k_dense_soft block fits next to a k_pair CTA (opt-in; measured slower,
// DESIGN.md section 5.2).
int launch_dense_soft(const PairArgs& a, bool write_grad, int exclude_smem, void* stream) {
  if (static_cast<long long>(a.t_max) * a.B == 0) return cudaSuccess;
  return launch_dense_rows<true>(a, write_grad, exclude_smem, stream);
}

int launch_dense_patch(const PairArgs& a, void* stream) {
  const long long rows = static_cast<long long>(a.t_max) * a.B;
  if (rows == 0 || a.grad == nullptr) return cudaSuccess;
  k_dense_patch<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

int launch_finalize(const PairArgs& a, void* stream) {
  if (a.B == 0) return cudaSuccess;
  k_finalize<<<a.B, kFinalizeThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

int launch_loss_sum(const float* costs, int B, double* out2, void* stream) {
  k_loss_sum<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(costs, B, out2);
  return cudaGetLastError();
}

}  // namespace ds2ctc
