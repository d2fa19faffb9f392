// ctc_lattice.cu -- full CTC lattice export on sm_100a.
//
// Reference: asr::ctc::ctc_lattice (proj/src/ctc.cpp:145-169; CtcLattice,
// proj/include/asr/ctc.hpp:55-60): alpha (forward_column, ctc.cpp:109-124)
// and the emission-exclusive beta (backward_column, ctc.cpp:126-143) over
// log_softmax_rows(frame_logits), every cell of every column, plus log p
// (final_log_prob, ctc.cpp:81-87). This is the debug / verification path of
// the pair kernel's column-parallel scheme (the cancellation property of
// test_ctc.cpp:172-199), so it follows the reference operation by operation
// in fp64: log_sum_exp_guarded (ctc.hpp:30-35) with the same -inf discard
// rule and operand order, one thread per frame for each row's lse.
//
// Two CTAs per utterance (alpha, beta) run concurrently; threads over the
// S = 2L+1 rows, the previous column in shared memory, every column written
// to the caller's [S][T] matrices (row-major, the reference Matrix(s, t)).
#include <cuda_runtime.h>

#include <cstdint>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

constexpr int kLatticeThreads = 256;

__device__ __forceinline__ double lse_guarded(double a, double b) {  // ctc.hpp:30-35
  const double NEG = -__builtin_huge_val();
  if (a == NEG) return b;
  if (b == NEG) return a;
  if (a < b) {
    const double t = a;
    a = b;
    b = t;
  }
  return a + log1p(exp(b - a));
}

__global__ void __launch_bounds__(kLatticeThreads) k_lattice(LatticeArgs a) {
  extern __shared__ __align__(16) unsigned char lsm[];
  const int b = blockIdx.x >> 1;
  const bool fwd = (blockIdx.x & 1) == 0;
  const ViterbiDesc d = a.desc[b];
  const int tid = threadIdx.x;
  const int T = d.T, S = 2 * d.L + 1;
  double* lse = reinterpret_cast<double*>(lsm);  // [T]
  double* c0 = lse + T;                           // [S]
  double* c1 = c0 + S;                            // [S]
  int* aug = reinterpret_cast<int*>(c1 + S);      // [S]
  const size_t rs = static_cast<size_t>(a.B) * a.A;
  const float* xb = a.x + static_cast<size_t>(b) * a.A;
  double* out = (fwd ? a.alpha : a.beta) + d.bp_off;  // [S][T]
  const double NEG = -__builtin_huge_val();

  for (int s = tid; s < S; s += kLatticeThreads) aug[s] = (s & 1) ? a.labels[d.lab_off + (s >> 1)] : a.blank;
  for (int t = tid; t < T; t += kLatticeThreads) {  // log_softmax_rows (ctc.cpp:24-37)
    const float* row = xb + static_cast<size_t>(t) * rs;
    double mx = row[0];
    for (int c = 1; c < a.A; ++c) mx = fmax(mx, static_cast<double>(row[c]));
    double sum = 0.0;
    for (int c = 0; c < a.A; ++c) sum += exp(static_cast<double>(row[c]) - mx);
    lse[t] = mx + log(sum);
  }
  __syncthreads();
  auto lp = [&](int t, int s) { return static_cast<double>(xb[static_cast<size_t>(t) * rs + aug[s]]) - lse[t]; };
  auto skip_ok = [&](int s) { return s >= 2 && aug[s] != a.blank && aug[s] != aug[s - 2]; };
  double* prev = c0;
  double* cur = c1;
  if (fwd) {
    for (int t = 0; t < T; ++t) {
      for (int s = tid; s < S; s += kLatticeThreads) {
        double v;
        if (t == 0) {
          v = s < 2 ? lp(0, s) : NEG;
        } else {
          double acc = prev[s];
          if (s >= 1) acc = lse_guarded(acc, prev[s - 1]);
          if (skip_ok(s)) acc = lse_guarded(acc, prev[s - 2]);
          v = acc == NEG ? NEG : acc + lp(t, s);
        }
        cur[s] = v;
        out[static_cast<size_t>(s) * T + t] = v;
      }
      __syncthreads();
      double* tmp = prev;
      prev = cur;
      cur = tmp;
    }
    if (tid == 0) {  // final_log_prob (ctc.cpp:81-87)
      double lpz = NEG;
      if (S >= 2) lpz = lse_guarded(lpz, prev[S - 2]);
      a.log_prob[b] = lse_guarded(lpz, prev[S - 1]);
    }
  } else {
    for (int t = T - 1; t >= 0; --t) {
      for (int s = tid; s < S; s += kLatticeThreads) {
        double v;
        if (t == T - 1) {
          v = s >= S - 2 ? 0.0 : NEG;
        } else {
          double acc = prev[s] == NEG ? NEG : prev[s] + lp(t + 1, s);
          if (s + 1 < S && prev[s + 1] != NEG) acc = lse_guarded(acc, prev[s + 1] + lp(t + 1, s + 1));
          if (s + 2 < S && skip_ok(s + 2) && prev[s + 2] != NEG) acc = lse_guarded(acc, prev[s + 2] + lp(t + 1, s + 2));
          v = acc;
        }
        cur[s] = v;
        out[static_cast<size_t>(s) * T + t] = v;
      }
      __syncthreads();
      double* tmp = prev;
      prev = cur;
      cur = tmp;
    }
  }
}

}  // namespace

size_t lattice_smem_bytes(int T, int L) {
  const size_t S = 2 * static_cast<size_t>(L) + 1;
  return 8 * (static_cast<size_t>(T) + 2 * S) + 4 * S;
}

int launch_lattice(const LatticeArgs& a, size_t smem, void* stream) {
  if (a.B == 0) return cudaSuccess;
  static int configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t err =
        cudaFuncSetAttribute(k_lattice, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBudget));
    if (err != cudaSuccess) return err;
    if (dev >= 0 && dev < 64) configured[dev] = 1;
  }
  k_lattice<<<2 * a.B, kLatticeThreads, smem, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

}  // namespace ds2ctc
