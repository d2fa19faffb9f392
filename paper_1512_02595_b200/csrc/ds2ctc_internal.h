// ds2ctc_internal.h -- shared host/device definitions of the CTC pipeline.
//
// Pipeline per ds2ctc_compute_loss call (all on the caller's stream):
//   H2D   one packed metadata blob (UttDesc[], launch order, labels, key CSR)
//   K1    rowstats   : per frame (max, log-sum-exp) of the logits   (HBM-bound)
//   K2/3  pair chain : per utterance a 2-CTA cluster, alpha forward || beta
//                      backward, meet at the midpoint, then each CTA fuses
//                      occupancy + gradient for its half             (latency-bound)
//   K4    dense      : large alphabets only -- one coalesced pass writing
//                      softmax - occupancy                             (HBM-bound)
#pragma once

#include <cstddef>
#include <cstdint>

namespace ds2ctc {

constexpr int kMaxStates = 4095;   // == DS2CTC_MAX_STATES
constexpr int kFusedMaxAlphabet = 1024;
constexpr size_t kAlign = 256;

// Per-utterance descriptor, computed on the host, read by every kernel.
struct alignas(16) UttDesc {
  int T;         // input length (frames)
  int L;         // label length
  int S;         // 2L+1
  int status;    // 0 = run, 1 = infeasible (T < min_frames), 2 = trivial (T == 0, L == 0: cost 0)
  int lab_off;   // offset into labels[]
  int nkey;      // key slots: slot 0 = blank, slots 1..nkey-1 = distinct non-blank symbols
  int key_off;   // offset into key_char[] / key_start[] (key_start has nkey+1 entries at key_off+b)
  int row_off;   // offset into key_rows[] (odd lattice rows grouped by slot)
  long long store_off;  // offset (doubles) into the half-lattice store: S * (T + 1) doubles
  long long occ_off;    // offset (floats) into the compact occupancy rows (dense path): T * nkey
  int tm;        // meet-in-the-middle frame
  int pad0, pad1, pad2;
};
static_assert(sizeof(UttDesc) == 64, "UttDesc layout");

// Offsets (bytes) of the workspace regions; a pure function of the lengths.
struct Layout {
  size_t desc, order, labels, key_char, key_start, key_rows, meta_end;  // metadata blob (int32 words)
  size_t stats;   // float2 [T_max * B]
  size_t store;   // double [sum S_b (T_b + 1)]
  size_t occ;     // float  [sum T_b (L_b + 1)] (dense path only)
  size_t logz;    // double [B]
  size_t total;
  int t_max;
  long long sum_L;
};

inline size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

inline Layout make_layout(const int* label_lengths, const int* input_lengths, int A, int B) {
  Layout lay{};
  long long sum_L = 0, store = 0, occ = 0;
  int t_max = 0;
  for (int b = 0; b < B; ++b) {
    long long L = label_lengths[b], T = input_lengths[b];
    sum_L += L;
    store += (2 * L + 1) * (T + 1);
    occ += T * (L + 1);
    if (T > t_max) t_max = static_cast<int>(T);
  }
  size_t off = 0;
  lay.desc = off;      off += sizeof(UttDesc) * B;
  lay.order = off;     off += sizeof(int) * B;
  lay.labels = off;    off += sizeof(int) * sum_L;
  lay.key_char = off;  off += sizeof(int) * (sum_L + B);
  lay.key_start = off; off += sizeof(int) * (sum_L + 2 * B);
  lay.key_rows = off;  off += sizeof(int) * sum_L;
  lay.meta_end = off;
  off = align_up(off);
  lay.stats = off;     off = align_up(off + sizeof(float) * 2 * static_cast<size_t>(t_max) * B);
  lay.store = off;     off = align_up(off + sizeof(double) * static_cast<size_t>(store));
  lay.occ = off;
  if (A > kFusedMaxAlphabet) off += sizeof(float) * static_cast<size_t>(occ);
  off = align_up(off);
  lay.logz = off;      off = align_up(off + sizeof(double) * B);
  lay.total = off;
  lay.t_max = t_max;
  lay.sum_L = sum_L;
  return lay;
}

// Kernel launch parameters (device pointers into the caller's buffers/workspace).
struct ChainArgs {
  const float* x;        // [T_max][B][A]
  float* grad;           // [T_max][B][A] or nullptr
  float* costs;          // [B]
  const UttDesc* desc;
  const int* order;
  const int* labels;
  const int* key_char;
  const int* key_start;
  const int* key_rows;
  const float2* stats;   // [T_max][B]
  double* store;
  float* occ;            // dense path compact occupancy rows, nullptr when fused
  double* logz;          // [B] log2-domain log Z (-inf when infeasible)
  int t_max, B, A, blank;
  int nthreads;          // CTA size of the chain kernel
  int cells;             // cells per thread (K)
};

// Launchers (ctc_kernels.cu). Return cudaError_t as int.
int launch_rowstats(const ChainArgs& a, void* stream);
int launch_chain(const ChainArgs& a, void* stream);
int launch_dense(const ChainArgs& a, void* stream);

}  // namespace ds2ctc
