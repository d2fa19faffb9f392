// ctc_viterbi.cu -- CTC forced alignment on sm_100a.
//
// Reference: asr::ctc::viterbi_align (proj/src/ctc.cpp:327-370; declared
// proj/include/asr/ctc.hpp:97-101): the max-plus recursion over the same
// blank-extended lattice as the forward pass, with backpointers, on
// log_softmax_rows(frame_logits) (ctc.cpp:24-37). Ties keep the largest
// predecessor row (stay > advance by one > skip, strict '>' as in the
// reference) and the final row prefers the terminal label over the terminal
// blank only if strictly better. The alignment is an index sequence, so it
// must be bit-identical to the reference: the scores are carried in fp64
// with the reference's operation order (lp = x - lse stored per cell, then
// best + lp), and each frame's lse is one thread's sequential max / sum exp
// / log over the row, exactly as log_softmax_rows.
//
// One CTA per utterance; threads over the S = 2L+1 lattice rows; the two
// score columns live in shared memory, backpointers (2 bits used per cell,
// one byte stored) in the workspace; thread 0 walks them back.
#include <cuda_runtime.h>

#include <cstdint>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

constexpr int kViterbiThreads = 256;

__global__ void __launch_bounds__(kViterbiThreads) k_viterbi(ViterbiArgs a) {
  extern __shared__ __align__(16) unsigned char vsm[];
  const int b = blockIdx.x;
  const ViterbiDesc d = a.desc[b];
  const int tid = threadIdx.x;
  int* out = a.align + static_cast<size_t>(b) * a.t_max;
  for (int t = d.T + tid; t < a.t_max; t += kViterbiThreads) out[t] = -1;  // padded frames
  if (d.status != 0) {  // infeasible for T (ctc.cpp:328 throws): no alignment
    for (int t = tid; t < d.T; t += kViterbiThreads) out[t] = -1;
    if (tid == 0) a.status[b] = 1;
    return;
  }
  const int T = d.T, S = 2 * d.L + 1;
  double* lse = reinterpret_cast<double*>(vsm);                 // [T]
  double* col0 = lse + T;                                         // [S]
  double* col1 = col0 + S;                                        // [S]
  int* aug = reinterpret_cast<int*>(col1 + S);                    // [S]
  const size_t rs = static_cast<size_t>(a.B) * a.A;               // frame stride of [T][B][A]
  const float* xb = a.x + static_cast<size_t>(b) * a.A;
  unsigned char* bp = a.bp + d.bp_off;                            // [T][S]

  for (int s = tid; s < S; s += kViterbiThreads) aug[s] = (s & 1) ? a.labels[d.lab_off + (s >> 1)] : a.blank;
  // log_softmax_rows (ctc.cpp:24-37), one frame per thread in the reference's order
  for (int t = tid; t < T; t += kViterbiThreads) {
    const float* row = xb + static_cast<size_t>(t) * rs;
    double mx = row[0];
    for (int c = 1; c < a.A; ++c) mx = fmax(mx, static_cast<double>(row[c]));
    double sum = 0.0;
    for (int c = 0; c < a.A; ++c) sum += exp(static_cast<double>(row[c]) - mx);
    lse[t] = mx + log(sum);
  }
  __syncthreads();
  const double NEG = -__builtin_huge_val();
  for (int s = tid; s < S; s += kViterbiThreads)
    col0[s] = s < 2 ? static_cast<double>(xb[aug[s]]) - lse[0] : NEG;
  __syncthreads();
  double* prev = col0;
  double* cur = col1;
  for (int t = 1; t < T; ++t) {
    const float* row = xb + static_cast<size_t>(t) * rs;
    const double lt = lse[t];
    unsigned char* bpt = bp + static_cast<size_t>(t) * S;
    for (int s = tid; s < S; s += kViterbiThreads) {
      double best = prev[s];
      unsigned char from = 0;  // stay
      if (s >= 1 && prev[s - 1] > best) {
        best = prev[s - 1];
        from = 1;
      }
      // skip_allowed (ctc.cpp:41-43)
      if (s >= 2 && aug[s] != a.blank && aug[s] != aug[s - 2] && prev[s - 2] > best) {
        best = prev[s - 2];
        from = 2;
      }
      if (best == NEG) {
        cur[s] = NEG;
        from = 3;
      } else {
        const double lp = static_cast<double>(row[aug[s]]) - lt;
        cur[s] = best + lp;
      }
      bpt[s] = from;
    }
    __syncthreads();
    double* tmp = prev;
    prev = cur;
    cur = tmp;
  }
  if (tid == 0) {
    int end = S - 1;
    if (S >= 2 && prev[S - 2] > prev[end]) end = S - 2;
    if (prev[end] == NEG) {  // no path of nonzero probability (ctc.cpp:361)
      for (int t = 0; t < T; ++t) out[t] = -1;
      a.status[b] = 1;
    } else {
      int s = end;
      for (int t = T - 1; t >= 0; --t) {
        out[t] = aug[s];
        if (t > 0) s -= bp[static_cast<size_t>(t) * S + s];
      }
      a.status[b] = 0;
    }
  }
}

}  // namespace

size_t viterbi_smem_bytes(int T, int L) {
  const size_t S = 2 * static_cast<size_t>(L) + 1;
  return 8 * (static_cast<size_t>(T) + 2 * S) + 4 * S;
}

int launch_viterbi(const ViterbiArgs& a, size_t smem, void* stream) {
  if (a.B == 0) return cudaSuccess;
  static int configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t err =
        cudaFuncSetAttribute(k_viterbi, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBudget));
    if (err != cudaSuccess) return err;
    if (dev >= 0 && dev < 64) configured[dev] = 1;
  }
  k_viterbi<<<a.B, kViterbiThreads, smem, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

}  // namespace ds2ctc
