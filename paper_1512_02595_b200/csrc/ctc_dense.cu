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
constexpr int kDenseThreads = 256;
constexpr int kDenseVec = 8;  // float4 per thread in registers -> A <= 8192 on the vector path

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

__global__ void __launch_bounds__(kDenseThreads) k_dense(PairArgs a, int write_grad) {
  __shared__ float sh[32];
  const int row = blockIdx.x;
  const int t = row / a.B;
  const int b = row - t * a.B;
  const UttDesc u = a.desc[b];
  const int A = a.A;
  const int tid = threadIdx.x;
  float* gr = write_grad ? a.grad + static_cast<size_t>(row) * A : nullptr;
  const float* xr = a.x + static_cast<size_t>(row) * A;
  const bool live = u.status == 0 && t < u.T && a.logz[b] != -__builtin_huge_val();
  if (!live) {
    if (gr)
      for (int c = tid; c < A; c += kDenseThreads) gr[c] = 0.f;
    return;
  }
  const bool vec = (A & 3) == 0 && A <= kDenseVec * kDenseThreads * 4;
  float m, ls;
  if (vec) {  // the row stays in registers: one HBM read, one HBM write
    const int n4 = A >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(xr);
    float4 v[kDenseVec];
    m = -__builtin_huge_valf();
#pragma unroll
    for (int j = 0; j < kDenseVec; ++j) {
      const int q = tid + j * kDenseThreads;
      v[j] = q < n4 ? ldg_stream(x4 + q) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      m = fmaxf(m, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
    }
    m = block_max(m, sh);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kDenseVec; ++j)
      s += (__expf(v[j].x - m) + __expf(v[j].y - m)) + (__expf(v[j].z - m) + __expf(v[j].w - m));
    s = block_sum(s, sh);
    ls = logf(s);
    if (gr) {
      float4* g4 = reinterpret_cast<float4*>(gr);
      const float off = m + ls;
#pragma unroll
      for (int j = 0; j < kDenseVec; ++j) {
        const int q = tid + j * kDenseThreads;
        if (q < n4)
          stg_stream(g4 + q, make_float4(__expf(v[j].x - off), __expf(v[j].y - off), __expf(v[j].z - off),
                                         __expf(v[j].w - off)));
      }
    }
  } else {  // generic: two passes (the second hits L1/L2)
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
  if (!gr) return;
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

// The HBM pass split in two so that its bulk overlaps k_pair (which leaves the
// memory system idle for ~110 us at the Mandarin shape, while its one CTA
// per SM leaves room for more):
//  k_dense_soft  -- needs nothing from k_pair: per (t, b) row the max and the
//                   log-sum-exp (log_softmax_rows, ctc.cpp:24-37) and the
//                   softmax row written to the gradient, exp evaluated once
//                   per element (kept in registers between the sum and the
//                   store). Runs on a forked stream concurrently with k_pair.
//  k_dense_patch -- after k_pair: subtract the occupancies at the <= L + 1
//                   key columns of each row (grad_column, ctc.cpp:69-79), and
//                   zero the rows of utterances whose lattice has no mass.
__global__ void __launch_bounds__(kDenseThreads) k_dense_soft(PairArgs a, int write_grad) {
  __shared__ float sh[32];
  const int row = blockIdx.x;
  const int t = row / a.B;
  const int b = row - t * a.B;
  const UttDesc u = a.desc[b];
  const int A = a.A;
  const int tid = threadIdx.x;
  float* gr = write_grad ? a.grad + static_cast<size_t>(row) * A : nullptr;
  const float* xr = a.x + static_cast<size_t>(row) * A;
  if (!(u.status == 0 && t < u.T)) {
    if (gr)
      for (int c = tid; c < A; c += kDenseThreads) gr[c] = 0.f;
    return;
  }
  const bool vec = (A & 3) == 0 && A <= kDenseVec * kDenseThreads * 4;
  float m, ls;
  if (vec) {  // the row stays in registers: one HBM read, one HBM write
    const int n4 = A >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(xr);
    float4 v[kDenseVec];
    m = -__builtin_huge_valf();
#pragma unroll
    for (int j = 0; j < kDenseVec; ++j) {
      const int q = tid + j * kDenseThreads;
      v[j] = q < n4 ? ldg_stream(x4 + q) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      m = fmaxf(m, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
    }
    m = block_max(m, sh);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kDenseVec; ++j) {
      v[j] = make_float4(__expf(v[j].x - m), __expf(v[j].y - m), __expf(v[j].z - m), __expf(v[j].w - m));
      s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
    s = block_sum(s, sh);
    ls = logf(s);
    if (gr) {
      float4* g4 = reinterpret_cast<float4*>(gr);
      const float inv = 1.f / s;
#pragma unroll
      for (int j = 0; j < kDenseVec; ++j) {
        const int q = tid + j * kDenseThreads;
        if (q < n4) stg_stream(g4 + q, make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv));
      }
    }
  } else {  // generic: two passes (the second hits L1/L2)
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

// costs[b] = sum_t lse_t - log Z (natural log), one warp per utterance.
// log Z = log Z' + sum_t mk_t, with log Z' (log2 units) from k_pair.
__global__ void k_finalize(PairArgs a) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= a.B) return;
  const UttDesc u = a.desc[b];
  if (u.status != 0) {
    if (lane == 0) a.costs[b] = u.status == 2 ? 0.f : __builtin_huge_valf();
    return;
  }
  const double lz = a.logz[b];
  double acc = 0.0;
  for (int t = lane; t < u.T; t += 32) {
    const float2 v = a.lse[static_cast<size_t>(t) * a.B + b];
    acc += static_cast<double>(v.x) + static_cast<double>(v.y);
  }
  acc = warp_sum_d(acc);
  // k_pair ran on frames shifted by mk_t and left -sum_t mk_t in part[2b], part[2b+1].
  if (lane == 0)
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
    for (int t = lane; t < u.T; t += 32) {
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
  const long long rows = static_cast<long long>(a.t_max) * a.B;
  if (rows == 0) return cudaSuccess;
  k_dense<<<static_cast<unsigned>(rows), kDenseThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, write_grad ? 1 : 0);
  return cudaGetLastError();
}

int launch_dense_soft(const PairArgs& a, bool write_grad, void* stream) {
  const long long rows = static_cast<long long>(a.t_max) * a.B;
  if (rows == 0) return cudaSuccess;
  k_dense_soft<<<static_cast<unsigned>(rows), kDenseThreads, 0, static_cast<cudaStream_t>(stream)>>>(a,
                                                                                                    write_grad ? 1 : 0);
  return cudaGetLastError();
}

int launch_dense_patch(const PairArgs& a, void* stream) {
  const long long rows = static_cast<long long>(a.t_max) * a.B;
  if (rows == 0 || a.grad == nullptr) return cudaSuccess;
  k_dense_patch<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

int launch_finalize(const PairArgs& a, void* stream) {
  if (a.B == 0) return cudaSuccess;
  k_finalize<<<(a.B + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

int launch_loss_sum(const float* costs, int B, double* out2, void* stream) {
  k_loss_sum<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(costs, B, out2);
  return cudaGetLastError();
}

}  // namespace ds2ctc
