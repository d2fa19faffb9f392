// ds2ctc_internal.h -- shared host/device definitions of the CTC pipeline.
//
// Per ds2ctc_compute_loss call (all on the caller's stream):
//   H2D    one packed metadata blob (UttDesc[], launch order, labels, key CSR)
//   pair   k_pair: per utterance a 2-CTA cluster, alpha forward || beta
//          backward over the RAW logits, meeting at frame tm = (T-1)/2; each
//          CTA then streams its half of gamma = alpha+beta into occupancies.
//          Small alphabets (A <= kFusedMaxAlphabet): the same kernel also
//          computes the per-frame log-softmax statistics, the gradient rows
//          softmax - occupancy and the costs -> ONE launch per call.
//   dense  large alphabets only: one coalesced pass per frame computing the
//          log-sum-exp and writing softmax - occupancy (key chars only)
//   final  large alphabets only: costs = sum_t lse_t - log Z
#pragma once

#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define DS2CTC_HD __host__ __device__
#else
#define DS2CTC_HD
#endif

namespace ds2ctc {

constexpr int kMaxStates = 4095;  // == DS2CTC_MAX_STATES
constexpr int kFusedMaxAlphabet = 128;
constexpr int kMaxThreads = 384;  // <= 10 chain warps (K = 8, L <= 2047) + service + gradient warps
constexpr size_t kAlign = 256;
constexpr size_t kSmemBudget = 220 * 1024;
// Two CTAs per SM (the dual build for multi-wave batches): 228 KB per SM,
// 1 KB reserved per CTA.
constexpr size_t kSmemBudgetDual = 113 * 1024;

// Per-utterance descriptor, computed on the host, read by every kernel.
struct alignas(16) UttDesc {
  int T;          // input length (frames)
  int L;          // label length
  int S;          // 2L+1
  int status;     // 0 = run, 1 = infeasible (T < min_frames), 2 = trivial (T == 0, L == 0: cost 0)
  int lab_off;    // offset into labels[] (also into key_pos[])
  int nkey;       // key slots: slot 0 = blank, slots 1.. = distinct non-blank symbols ascending
  int key_off;    // offset into key_char[] (packed); key_start has nkey+1 entries at key_off + b
  int col_w;      // floats per stored lattice column: roundup4(S) + roundup4(chain warps)
  long long store_off;  // offset (floats) into the half-lattice store: col_w * (T + 1)
  long long occ_off;    // offset (floats) into the compact occupancy rows (split path): T * nkey
  int tm;         // meet-in-the-middle frame
  int pad0, pad1, pad2;
};
static_assert(sizeof(UttDesc) == 64, "UttDesc layout");

DS2CTC_HD inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// Floats per emission row: the staged symbols, the sentinel column (index SW)
// and padding to an odd stride (rows indexed by frame are bank-conflict free).
DS2CTC_HD inline int emis_stride(int SW) { return (SW + 1) | 1; }

// Launch geometry shared by every utterance of one call.
struct Geometry {
  int K;          // label pairs per chain thread
  int nchain;     // chain warps (max over the batch)
  int P;          // epoch length (steps between CTA barriers)
  int SW;         // staged symbols per frame: A (fused) or max nkey (split)
  int max_L;
  int fused;
  int dual;       // 1: two clusters per SM pair (k_pair<K, 2>, <= kSmemBudgetDual)
  // shared-memory carve-up (bytes, 16-aligned)
  int off_xraw, off_emis, off_lse, off_el, off_occ, off_ring, off_meta, off_red;
  int ring_depth; // halo refresh ring entries per chain warp
  int off_cb;     // column buffer [2][P][cw_max] floats (TMA bulk stores / loads of lattice columns)
  int off_mbar;   // two mbarriers (one per column-buffer half)
  int off_flag;   // poisoned-frame flags: [0] this CTA's phase-1 frames, [1] written by the partner at the meet
  int off_nrm;    // [2][column_threads(max_L)] per-thread frame mass of each phase-2 epoch's sampled column
  int xstride;    // floats per xraw row (odd)
  int estride;    // floats per occupancy (el) row (odd)
  int cw_max;     // floats per stored column (max over batch)
  int ostride;    // floats per occ scratch row (odd)
  int smem;       // total bytes
};

// Chain warps: 32 lanes, of which kHaloLanes recompute the upstream warp's
// edge lanes (refreshed every halo_steps(K) steps) and kOwnedLanes own cells.
constexpr int kHaloLanes = 4;
constexpr int kOwnedLanes = 32 - kHaloLanes;
// The halo absorbs the wrong outer neighbour for 2*kHaloLanes*K rows, i.e.
// kHaloLanes*K steps (the recursion moves 2 rows per step).
DS2CTC_HD inline int halo_steps(int K) { return kHaloLanes * K < 16 ? kHaloLanes * K : 16; }
DS2CTC_HD inline int column_threads(int L, int K) { return (L + 1 + K - 1) / K; }
DS2CTC_HD inline int chain_warps_for(int L, int K) { return (column_threads(L, K) + kOwnedLanes - 1) / kOwnedLanes; }

// Label pairs per chain thread. At most three chain warps while K <= 8, so
// the service warp keeps an SM sub-partition (SMSP) of its own; each pair
// costs 5 MUFU ops per step, so K also bounds the per-SMSP MUFU load.
constexpr int kPairChoices[] = {1, 2, 3, 4, 6, 8};
inline int pick_K(int max_L) {
  const int pairs = max_L + 1;
  for (int K : kPairChoices)
    if (pairs <= 3 * kOwnedLanes * K) return K;
  return 8;
}

// Stored half-lattice column, warp-blocked: chain warp w owns a block of
// (2K + 1) x 32 words; lane l's q-th slot (q < 2K) is word q * 32 + l of the
// block and its fp32 offset word 2K * 32 + l (forward: slot = cell s;
// backward: slot = s + 1). The strides between one lane's words are compile-
// time (one base register + immediates per step) and consecutive lanes touch
// consecutive words, so neither the owning warp's per-step stores nor the
// partner's phase-2 reads have shared-memory bank conflicts (the round-1
// thread-major layout gave 2K-way conflicts on the partner reads,
// profiles/r02_bank_conflicts.txt). Thread j of direction d sits in warp
// j / 28 at lane j % 28 (+ the 4 halo lanes first when d = 0, forward).
DS2CTC_HD inline int column_block(int K) { return (2 * K + 1) * 32; }
DS2CTC_HD inline int column_width(int L, int K) { return chain_warps_for(L, K) * column_block(K); }
DS2CTC_HD inline int thread_lane(int j, int dir) { return j % kOwnedLanes + (dir == 0 ? kHaloLanes : 0); }
// Word of stored slot q of chain thread j (direction dir's layout); q == 2K is its offset.
DS2CTC_HD inline int column_word(int j, int q, int K, int dir) {
  return (j / kOwnedLanes) * column_block(K) + q * 32 + thread_lane(j, dir);
}
DS2CTC_HD inline int column_slot_word(int slot, int K, int dir) { return column_word(slot / (2 * K), slot % (2 * K), K, dir); }
// Occupancy rows (phase 2): each label cell's occupancy at its position's
// slot-sorted rank (word L is the spare of cells without a label), so the
// gradient warp sums each key slot as one contiguous run.

// max_L_all: the longest label of the whole batch (it fixes K and hence the
// stored column layout, see make_layout); max_L: the longest that runs.
inline Geometry make_geometry(int max_L_all, int max_L, int max_nkey, int A, bool fused,
                              size_t budget = kSmemBudget) {
  Geometry g{};
  g.K = pick_K(max_L_all);
  g.nchain = chain_warps_for(max_L, g.K);
  g.max_L = max_L;
  g.fused = fused ? 1 : 0;
  g.SW = fused ? A : max_nkey;
  g.cw_max = column_width(max_L_all, g.K);
  for (int P = 32; P >= 2; P /= 2) {
    g.P = P;
    g.xstride = g.SW | 1;
    g.estride = (max_L + 1) | 1;  // slot-sorted label positions + a spare word
    g.ostride = max_nkey | 1;
    int off = 0;
    auto take = [&](int bytes) {
      int o = off;
      off += round_up(bytes, 16);
      return o;
    };
    const int RX = 4 * P;
    g.off_xraw = take(4 * RX * g.xstride);
    g.off_emis = take(4 * 2 * P * emis_stride(g.SW));  // + a sentinel column for cells that do not exist
    g.off_lse = take(8 * RX);
    g.off_el = take(4 * 2 * P * g.estride);
    g.off_occ = take(4 * 2 * 32 * g.ostride);  // double-buffered: label sums of epoch e-1 || gradient rows of e-2
    g.ring_depth = 4;  // a power of two >= 2 * (P / halo_steps + 2): the slot is a mask, not a division
    while (g.ring_depth < 2 * (P / halo_steps(g.K) + 2)) g.ring_depth *= 2;
    g.off_ring = take(8 * g.nchain * g.ring_depth * kHaloLanes * (2 * g.K + 1));
    g.off_cb = take(4 * 2 * P * g.cw_max);
    g.off_mbar = take(16);
    g.off_nrm = take(4 * 2 * column_threads(max_L, g.K));
    // meta: labels (L+1), key_char (nkey), key_start (nkey+1), key_pos (L), slot of each label
    // position (L+1), symbol -> slot (A shorts, fused)
    g.off_meta = take(4 * (4 * max_L + 2 * max_nkey + 8) + (fused ? 2 * A : 0));
    g.off_red = take(2048);  // meet reductions (doubles per warp) and the drain's per-part totals (floats)
    g.off_flag = take(16);
    g.smem = off;
    if (static_cast<size_t>(off) <= budget) break;
  }
  return g;
}

// Offsets (bytes) of the workspace regions; a pure function of the lengths.
struct Layout {
  size_t desc, order, labels, key_char, key_start, key_pos, meta_end;  // metadata blob (int32 words)
  size_t store;   // float [sum col_w (T_b + 1)]
  size_t occ;     // float [sum T_b (L_b + 1)]   (split path)
  size_t lse;     // float2 [T_max * B]          (split path)
  size_t logz;    // double [B]
  size_t part;    // double [2B] per-CTA partial lse sums (fused path)
  size_t total;
  int t_max;
  long long sum_L;
};

inline size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

inline Layout make_layout(const int* label_lengths, const int* input_lengths, int A, int B) {
  Layout lay{};
  long long sum_L = 0, store = 0, occ = 0;
  int t_max = 0, max_L = 0;
  for (int b = 0; b < B; ++b) max_L = label_lengths[b] > max_L ? label_lengths[b] : max_L;
  const int K = pick_K(max_L);
  for (int b = 0; b < B; ++b) {
    long long L = label_lengths[b], T = input_lengths[b];
    sum_L += L;
    store += static_cast<long long>(column_width(static_cast<int>(L), K)) * (T + 1);
    occ += T * (L + 1);
    if (T > t_max) t_max = static_cast<int>(T);
  }
  const bool split = A > kFusedMaxAlphabet;
  size_t off = 0;
  lay.desc = off;      off += sizeof(UttDesc) * B;
  lay.order = off;     off += sizeof(int) * B;
  lay.labels = off;    off += sizeof(int) * sum_L;
  lay.key_pos = off;   off += sizeof(int) * sum_L;
  // key_char (sum nkey) then key_start (sum nkey + B), packed at run time from
  // here: only the used prefix of the blob is copied (nkey <= min(L+1, A))
  lay.key_char = off;  off += sizeof(int) * (sum_L + B);
  lay.key_start = off; off += sizeof(int) * (sum_L + 2 * B);
  lay.meta_end = off;
  off = align_up(off);
  lay.store = off;     off = align_up(off + sizeof(float) * static_cast<size_t>(store));
  lay.occ = off;       if (split) off = align_up(off + sizeof(float) * static_cast<size_t>(occ));
  lay.lse = off;       if (split) off = align_up(off + sizeof(float) * 2 * static_cast<size_t>(t_max) * B);
  lay.logz = off;      off = align_up(off + sizeof(double) * B);
  lay.part = off;      off = align_up(off + sizeof(double) * 2 * B);
  lay.total = off;
  lay.t_max = t_max;
  lay.sum_L = sum_L;
  return lay;
}

// Kernel arguments (device pointers into the caller's buffers / workspace).
struct PairArgs {
  const float* x;        // [T_max][B][A]
  float* grad;           // [T_max][B][A] or nullptr (cost only)
  float* costs;          // [B]
  const UttDesc* desc;
  const int* order;
  const int* labels;
  const int* key_char;
  const int* key_start;
  const int* key_pos;
  float* store;          // half-lattice columns
  float* occ;            // split path: compact occupancy rows
  float2* lse;           // split path: per-frame (max, log-sum-exp)
  double* logz;          // [B] log2-domain log Z (-inf when the lattice has zero mass)
  double* part;          // [2B] per-CTA partial sums of lse (fused path)
  int t_max, B, A, blank;
  int ld;  // frame stride of x / grad in utterances (B, or the caller's batch for a sub-batch view)
  Geometry g;
};

// Forced alignment (ctc_viterbi.cu; viterbi_align, ctc.cpp:327-370).
struct alignas(16) ViterbiDesc {
  int T, L, lab_off, status;  // status 1: T < min_frames or T == 0 (the reference throws)
  long long bp_off;           // byte offset of the utterance's [T][2L+1] backpointers
  long long pad;
};
static_assert(sizeof(ViterbiDesc) == 32, "ViterbiDesc layout");

struct ViterbiArgs {
  const float* x;  // [T_max][B][A]
  const ViterbiDesc* desc;
  const int* labels;
  unsigned char* bp;
  int* align;   // [B][T_max]: alignment symbols, -1 past T_b or without alignment
  int* status;  // [B]: 0 aligned, 1 infeasible / no path of nonzero probability
  int t_max, B, A, blank;
};

// Full lattice export (ctc_lattice.cu; ctc_lattice, ctc.cpp:145-169). The
// descriptor's bp_off is the utterance's cell offset into alpha / beta.
struct LatticeArgs {
  const float* x;  // [T_max][B][A]
  const ViterbiDesc* desc;
  const int* labels;
  double* alpha;     // sum_b S_b * T_b cells, utterance b row-major [S_b][T_b]
  double* beta;      // same layout (emission-exclusive beta)
  double* log_prob;  // [B]
  int t_max, B, A, blank;
};

struct ViterbiLayout {
  size_t desc, labels, bp, total;
  int t_max;
};

inline ViterbiLayout make_viterbi_layout(const int* label_lengths, const int* input_lengths, int B) {
  ViterbiLayout v{};
  long long sum_L = 0, bp = 0;
  for (int b = 0; b < B; ++b) {
    sum_L += label_lengths[b];
    bp += static_cast<long long>(input_lengths[b]) * (2LL * label_lengths[b] + 1);
    v.t_max = input_lengths[b] > v.t_max ? input_lengths[b] : v.t_max;
  }
  size_t off = 0;
  v.desc = off;
  off += sizeof(ViterbiDesc) * B;
  v.labels = off;
  off += sizeof(int) * static_cast<size_t>(sum_L);
  off = (off + kAlign - 1) / kAlign * kAlign;
  v.bp = off;
  off += static_cast<size_t>(bp);
  v.total = B > 0 ? (off + kAlign - 1) / kAlign * kAlign : 0;
  return v;
}

// Launchers (ctc_pair.cu / ctc_dense.cu / ctc_viterbi.cu). Return cudaError_t as int.
int launch_pair(const PairArgs& a, void* stream);
int launch_pair_k8(const PairArgs& a, void* stream);  // ctc_pair_k8.cu
int read_watchdog_k8(unsigned long long* out4);
int launch_dense(const PairArgs& a, bool write_grad, void* stream);
int launch_finalize(const PairArgs& a, void* stream);
int launch_dense_soft(const PairArgs& a, bool write_grad, int exclude_smem, void* stream);
int launch_dense_patch(const PairArgs& a, void* stream);
int launch_loss_sum(const float* costs, int B, double* out2, void* stream);

// Peer mailboxes of the fused scalar all-reduce (ctc_reduce.cu): this
// process's view (own buffer or CUDA IPC mapping) of every rank's mailbox.
constexpr int kMaxPeers = 8;
struct PeerMailboxes {
  void* peer[kMaxPeers];
  int rank, world;
};
int launch_loss_allreduce(const float* costs, int B, double* out2, const PeerMailboxes& mb, unsigned long long seq,
                          void* stream);
size_t mailbox_bytes(int world);
size_t vec_exchange_bytes(long long n);
int launch_vec_allreduce(float* data, long long n, const PeerMailboxes& pr, unsigned long long seq, void* stream);
int read_reduce_fault(unsigned long long* seq);
int read_watchdog(unsigned long long* out4);
size_t viterbi_smem_bytes(int T, int L);
// Output-FC backward on tcgen05 (fc_backward.cu; nn.cpp:874-899).
size_t fc_backward_workspace(int rows, int A, int H);
int fc_backward(const float* g, const float* x, const float* w, float* dw, float* db, float* dx, int rows, int A,
                int H, void* workspace, int sm_count, void* stream);
int launch_viterbi(const ViterbiArgs& a, size_t smem, void* stream);
size_t lattice_smem_bytes(int T, int L);
int launch_lattice(const LatticeArgs& a, size_t smem, void* stream);

}  // namespace ds2ctc
