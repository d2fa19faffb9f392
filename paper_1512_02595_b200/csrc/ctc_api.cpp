// ctc_api.cpp -- C-ABI of libds2ctc (include/ds2ctc.h): validation, per-call
// metadata (the reference's augment_label / min_frames / group_rows_by_key,
// ctc.cpp:47-66,91-107, done once per utterance on the host), workspace
// layout, and the kernel pipeline on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <numeric>
#include <utility>
#include <vector>

#include "ds2ctc.h"
#include "ds2ctc_internal.h"


namespace ds2ctc {
namespace {

// Pinned staging ring for the per-call metadata blob, one per (thread, device).
// A slot is reused only after the event recorded behind its last copy fired.
class Staging {
 public:
  ~Staging() {
    for (auto& s : slots_) {
      if (s.ev) cudaEventDestroy(s.ev);
      if (s.ptr) cudaFreeHost(s.ptr);
    }
  }
  // Returns a pinned buffer of at least `bytes`, or nullptr.
  void* acquire(size_t bytes, cudaEvent_t* ev_out) {
    Slot& s = slots_[next_];
    next_ = (next_ + 1) % kSlots;
    if (s.ev) cudaEventSynchronize(s.ev);
    if (s.cap < bytes) {
      if (s.ptr) cudaFreeHost(s.ptr);
      s.ptr = nullptr;
      s.cap = 0;
      size_t want = std::max<size_t>(bytes, 64 << 10);
      if (cudaMallocHost(&s.ptr, want) != cudaSuccess) return nullptr;
      s.cap = want;
    }
    if (!s.ev && cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    *ev_out = s.ev;
    return s.ptr;
  }

 private:
  // One slot per call (a length-split call packs its sub-batches' blobs into
  // one slot), so the host can run 8 calls ahead of the GPU. Growing a slot
  // is a cudaMallocHost, so the slots must be warm before any timed call:
  // few of them, reused round-robin.
  static constexpr int kSlots = 8;
  struct Slot {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
  };
  Slot slots_[kSlots];
  int next_ = 0;
};

Staging& staging_for_current_device() {
  thread_local std::map<int, Staging> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  return per_device[dev];
}

// Optional per-thread stage timing (ds2ctc_profile_enable / _read): a ring
// of event sets so timed calls never synchronise the host.
struct Profiler {
  int slots = 0;
  int device = -1;
  long long calls = 0;
  // 6 per slot: 0 start, 1 after k_pair, 2 after the dense pass, 3 end (all on
  // the caller's stream); 4, 5 around k_dense_soft on the side stream when the
  // dense pass overlaps k_pair (then the "dense" stage is that kernel alone)
  std::vector<cudaEvent_t> ev;
  std::vector<int> side;  // per slot: 1 when events 4, 5 were recorded
  void reset() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    ev.clear();
    calls = 0;
    device = -1;
  }
  bool ready(int dev) {
    if (slots <= 0) return false;
    if (device != dev || static_cast<int>(ev.size()) != 6 * slots) {
      reset();
      ev.assign(6 * slots, nullptr);
      side.assign(slots, 0);
      for (auto& e : ev)
        if (cudaEventCreate(&e) != cudaSuccess) return false;
      device = dev;
    }
    return calls < slots;
  }
  void mark(int i, cudaStream_t s) {
    cudaEventRecord(ev[6 * calls + i], s);
    if (i == 0) side[calls] = 0;
    if (i == 4) side[calls] = 1;
  }
  bool suspended = false;  // inside a length-split call: one record for the whole call
};

Profiler& profiler() {
  thread_local Profiler p;
  return p;
}

int min_frames(const int* label, int L) {  // ctc.cpp:102-107
  int needed = L;
  for (int i = 1; i < L; ++i)
    if (label[i] == label[i - 1]) ++needed;
  return needed;
}

ds2ctc_status validate(const int* label_lengths, const int* input_lengths, int A, int B, int blank,
                       const int* flat_labels) {
  if (B < 0 || A < 2 || blank < 0 || blank >= A) return DS2CTC_STATUS_INVALID_VALUE;
  if (B > 0 && (label_lengths == nullptr || input_lengths == nullptr)) return DS2CTC_STATUS_INVALID_VALUE;
  long long sum_L = 0;
  for (int b = 0; b < B; ++b) {
    if (label_lengths[b] < 0 || input_lengths[b] < 0) return DS2CTC_STATUS_INVALID_VALUE;
    if (2LL * label_lengths[b] + 1 > kMaxStates) return DS2CTC_STATUS_UNSUPPORTED;
    sum_L += label_lengths[b];
  }
  if (sum_L > 0 && flat_labels == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  for (long long i = 0; i < sum_L; ++i)
    if (flat_labels[i] < 0 || flat_labels[i] >= A) return DS2CTC_STATUS_INVALID_VALUE;
  return DS2CTC_STATUS_SUCCESS;
}

// Builds the metadata blob (int32 words laid out per Layout) into `blob`.
// Returns (max L, max nkey) over utterances that run the lattice.
// The key map is packed: key_char (sum nkey words) from lay.key_char, then
// key_start (sum nkey + B words) right after it; *key_start_off and
// *meta_used receive that offset and the bytes to copy.
std::pair<int, int> build_metadata(const Layout& lay, const int* flat_labels, const int* label_lengths,
                                   const int* input_lengths, int A, int B, int blank, std::vector<int32_t>& blob,
                                   size_t* key_start_off, size_t* meta_used) {
  blob.resize(lay.meta_end / sizeof(int32_t));  // every word below the used prefix is written
  auto* desc = reinterpret_cast<UttDesc*>(blob.data() + lay.desc / 4);
  int* order = blob.data() + lay.order / 4;
  int* labels = blob.data() + lay.labels / 4;
  int* key_char = blob.data() + lay.key_char / 4;
  thread_local std::vector<int> key_start_v;
  key_start_v.resize(static_cast<size_t>(lay.sum_L) + 2 * B + 1);
  int* key_start = key_start_v.data();
  int* key_pos = blob.data() + lay.key_pos / 4;
  if (lay.sum_L > 0) std::memcpy(labels, flat_labels, sizeof(int) * lay.sum_L);

  // Per-symbol scratch (hoisted out of thread-local storage for the loops):
  // a presence bitset over the alphabet (ascending symbol order by a word
  // scan) and counts, both cleared after each utterance.
  thread_local std::vector<uint64_t> bits_v;
  thread_local std::vector<int> cnt_v, next_v;
  const int nwords = (A + 63) / 64;
  if (static_cast<int>(cnt_v.size()) < A) {
    bits_v.assign(nwords, 0ull);
    cnt_v.assign(A, 0);
    next_v.assign(A, 0);
  }
  uint64_t* bits = bits_v.data();
  int* cnt = cnt_v.data();
  int* next = next_v.data();

  int max_L_all = 0;
  for (int b = 0; b < B; ++b) max_L_all = std::max(max_L_all, label_lengths[b]);
  const int K = pick_K(max_L_all);
  long long lab_off = 0, key_off = 0, store_off = 0, occ_off = 0;
  int max_L = 0, max_nkey = 1;
  for (int b = 0; b < B; ++b) {
    UttDesc& u = desc[b];
    const int T = input_lengths[b], L = label_lengths[b];
    const int* lab = flat_labels + lab_off;
    u.T = T;
    u.L = L;
    u.S = 2 * L + 1;
    u.status = T < min_frames(lab, L) ? 1 : (T == 0 ? 2 : 0);
    u.lab_off = static_cast<int>(lab_off);
    u.key_off = static_cast<int>(key_off);
    u.col_w = column_width(L, K);
    u.store_off = store_off;
    u.occ_off = occ_off;
    u.tm = T > 0 ? (T - 1) / 2 : 0;
    u.pad0 = u.pad1 = u.pad2 = 0;
    // Key groups (group_rows_by_key, ctc.cpp:47-66) over label positions:
    // slot 0 = blank (all even lattice rows, plus label positions whose symbol
    // is the blank id), slots 1.. = distinct non-blank symbols ascending,
    // positions ascending within a slot. Counting sort by symbol.
    int* kc = key_char + key_off;
    int* ks = key_start + key_off + b;
    int nkey = 1;
    kc[0] = blank;
    ks[0] = 0;
    int n_blank = 0;
    for (int i = 0; i < L; ++i) {
      const int sym = lab[i];
      if (sym == blank) {
        ++n_blank;
        continue;
      }
      bits[sym >> 6] |= 1ull << (sym & 63);
      ++cnt[sym];
    }
    ks[1] = n_blank;
    next[blank] = 0;
    int run = n_blank;
    for (int w = 0; w < nwords; ++w) {
      uint64_t x = bits[w];
      if (x == 0) continue;
      bits[w] = 0;
      do {
        const int sym = w * 64 + __builtin_ctzll(x);
        x &= x - 1;
        kc[nkey] = sym;
        next[sym] = run;
        run += cnt[sym];
        cnt[sym] = 0;
        ks[++nkey] = run;
      } while (x);
    }
    int* kp = key_pos + lab_off;
    for (int i = 0; i < L; ++i) kp[next[lab[i]]++] = i;
    u.nkey = nkey;
    if (u.status == 0) {
      max_L = std::max(max_L, L);
      max_nkey = std::max(max_nkey, nkey);
    }
    lab_off += L;
    key_off += nkey;
    store_off += static_cast<long long>(u.col_w) * (T + 1);
    occ_off += static_cast<long long>(T) * nkey;
  }
  // key_start right behind the used part of key_char
  *key_start_off = lay.key_char + sizeof(int) * static_cast<size_t>(key_off);
  std::memcpy(blob.data() + *key_start_off / 4, key_start, sizeof(int) * static_cast<size_t>(key_off + B));
  *meta_used = *key_start_off + sizeof(int) * static_cast<size_t>(key_off + B);
  // Longest first (the serial chain is T steps), so long pairs start in the first wave.
  std::iota(order, order + B, 0);
  std::stable_sort(order, order + B, [&](int x, int y) {
    const int tx = desc[x].status == 0 ? desc[x].T : -1;
    const int ty = desc[y].status == 0 ? desc[y].T : -1;
    return tx > ty;
  });
  return {max_L, max_nkey};
}

// DS2CTC_DENSE_OVERLAP=1: the large-alphabet HBM pass split into k_dense_soft
// (concurrently with k_pair, on a forked stream) + k_dense_patch, instead of
// one k_dense after k_pair. Opt-in: with the register-resident row evaluated
// once per element, the serial pass measures faster (Mandarin 329 vs 337 us
// per step, profiles/r02_dense_ab.txt): co-resident dense blocks slow the chains
// (k_pair 122 -> 127 us), fit only ~2 per k_pair SM, and the patch re-reads
// the key columns.
bool dense_overlap_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("DS2CTC_DENSE_OVERLAP");
    return v != nullptr && std::atoi(v) != 0;
  }();
  return on;
}

// Dynamic shared memory (unused) for k_dense_soft such that none of its
// blocks fits on an SM next to the resident k_pair CTA(s): the concurrent
// softmax pass then runs on the SMs k_pair leaves free and on each SM as soon
// as k_pair releases it, instead of sharing issue slots with the chains
// (co-resident, English-style chains slowed from 112 to 156 us at the
// Mandarin shape). 0 = no exclusion: k_pair already fills the SM, or the
// request would leave fewer than two dense blocks per SM on their own.
// Opt-in (DS2CTC_DENSE_EXCLUDE=1): measured slower, 370 vs 345 us per
// Mandarin step -- the 20 SMs k_pair leaves free move too little of the pass
// and the request caps the later full-GPU part at 4 blocks per SM
// (profiles/r02_dense_ab.txt).
int dense_exclusion_smem(const Geometry& g) {
  static const bool on = [] {
    const char* v = std::getenv("DS2CTC_DENSE_EXCLUDE");
    return v != nullptr && std::atoi(v) != 0;
  }();
  if (!on) return 0;
  int dev = 0, cap = 0, reserved = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&cap, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return 0;
  const int resident = g.dual ? 2 : 1;  // k_pair CTAs per SM
  const int left = cap - resident * (g.smem + reserved);
  const int x = ((left - reserved) / 16 + 1) * 16;  // x + reserved > left
  if (x <= 0 || x > optin || 2 * (x + reserved) > cap) return 0;
  return x;
}

struct OverlapStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool init() {
    if (side) return true;
    return cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
};

OverlapStreams& overlap_streams_for_current_device() {
  thread_local std::map<int, OverlapStreams> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  return per_device[dev];
}

int sm_count() {
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (n[dev] == 0 && cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n[dev] = 148;
  return n[dev];
}

// DS2CTC_DUAL: 0 = never two clusters per SM pair, 1 = whenever it fits.
// Default: a makespan estimate. A k_pair CTA runs ~T_b dependent steps, so
// one cluster per SM pair finishes the batch in about max(T_max, sum T / P)
// step times (P = SMs / 2 cluster slots, LPT order); two per SM pair double
// the slots but each chain shares its SMSPs and runs ~1.9x slower per step
// (edge1500, K = 4: 1468 vs 765 cycles per step, profiles/r02_dual.txt).
// Dual wins on uniform multi-wave batches (edge1500: 7.85 vs 8.17 ms) and
// loses when one long utterance bounds the batch anyway (SortaGrad, 128
// utterances per GPU: T_max 1500 vs sum T / 74 ~ 1340 -> 0.91 ms dual).
constexpr double kDualSlowdown = 1.9;
bool dual_mode(int B, const int* input_lengths) {
  static const int env = [] {
    const char* v = std::getenv("DS2CTC_DUAL");
    return v ? std::atoi(v) : -1;
  }();
  if (env == 0) return false;
  if (env > 0) return true;
  const int sms = sm_count();
  if (2 * B <= sms) return false;  // one wave: nothing to gain
  double sum = 0.0;
  int tmax = 0;
  for (int b = 0; b < B; ++b) {
    sum += input_lengths[b];
    tmax = std::max(tmax, input_lengths[b]);
  }
  const double slots = sms / 2;
  const double single = std::max(static_cast<double>(tmax), sum / slots);
  const double dual = kDualSlowdown * std::max(static_cast<double>(tmax), sum / (2.0 * slots));
  return dual < single;
}

ds2ctc_status run(const float* acts, float* grads, const int* flat_labels, const int* label_lengths,
                  const int* input_lengths, int A, int B, int blank, float* costs, void* workspace,
                  size_t workspace_bytes, bool check_ws, void* stream, int ld = 0,
                  unsigned char* pinned_slice = nullptr) {
  ds2ctc_status st = validate(label_lengths, input_lengths, A, B, blank, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (B == 0) return DS2CTC_STATUS_SUCCESS;
  const Layout lay = make_layout(label_lengths, input_lengths, A, B);
  if (costs == nullptr || workspace == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (lay.t_max > 0 && acts == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (check_ws && workspace_bytes < lay.total) return DS2CTC_STATUS_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign != 0) return DS2CTC_STATUS_INVALID_VALUE;

  thread_local std::vector<int32_t> blob;
  size_t key_start_off = 0, meta_used = 0;
  const auto mx =
      build_metadata(lay, flat_labels, label_lengths, input_lengths, A, B, blank, blob, &key_start_off, &meta_used);

  auto* ws = static_cast<unsigned char*>(workspace);
  auto s = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev = nullptr;
  void* pinned = pinned_slice != nullptr ? pinned_slice : staging_for_current_device().acquire(meta_used, &ev);
  if (pinned == nullptr) return DS2CTC_STATUS_MEMOPS_FAILED;
  std::memcpy(pinned, blob.data(), meta_used);
  if (cudaMemcpyAsync(ws, pinned, meta_used, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return DS2CTC_STATUS_MEMOPS_FAILED;
  if (ev != nullptr && cudaEventRecord(ev, s) != cudaSuccess) return DS2CTC_STATUS_MEMOPS_FAILED;

  const bool fused = A <= kFusedMaxAlphabet;
  PairArgs a{};
  a.x = acts;
  a.grad = grads;
  a.costs = costs;
  a.desc = reinterpret_cast<const UttDesc*>(ws + lay.desc);
  a.order = reinterpret_cast<const int*>(ws + lay.order);
  a.labels = reinterpret_cast<const int*>(ws + lay.labels);
  a.key_char = reinterpret_cast<const int*>(ws + lay.key_char);
  a.key_start = reinterpret_cast<const int*>(ws + key_start_off);
  a.key_pos = reinterpret_cast<const int*>(ws + lay.key_pos);
  a.store = reinterpret_cast<float*>(ws + lay.store);
  a.occ = fused ? nullptr : reinterpret_cast<float*>(ws + lay.occ);
  a.lse = fused ? nullptr : reinterpret_cast<float2*>(ws + lay.lse);
  a.logz = reinterpret_cast<double*>(ws + lay.logz);
  a.part = reinterpret_cast<double*>(ws + lay.part);
  a.t_max = lay.t_max;
  a.B = B;
  a.A = A;
  a.blank = blank;
  a.ld = ld > 0 ? ld : B;
  if (a.ld != B && !fused) return DS2CTC_STATUS_INVALID_VALUE;  // k_dense / k_finalize index rows as t*B+b
  int max_L_all = 0;
  for (int b = 0; b < B; ++b) max_L_all = std::max(max_L_all, label_lengths[b]);
  a.g = make_geometry(max_L_all, mx.first, mx.second, A, fused);
  if (static_cast<size_t>(a.g.smem) > kSmemBudget) return DS2CTC_STATUS_UNSUPPORTED;
  // Multi-wave batches (more clusters than SM pairs): two clusters per SM
  // pair when the geometry fits half the shared memory with epochs of >= 8
  // steps and <= 3 chain warps (K <= 4) -- the chains are latency-bound, so a
  // second resident utterance uses issue slots the first leaves idle.
  if (dual_mode(B, input_lengths) && a.g.K <= 4 && a.g.nchain <= 3) {
    const Geometry g2 = make_geometry(max_L_all, mx.first, mx.second, A, fused, kSmemBudgetDual);
    if (static_cast<size_t>(g2.smem) <= kSmemBudgetDual && g2.P >= 8) {
      a.g = g2;
      a.g.dual = 1;
    }
  }

  int dev = 0;
  cudaGetDevice(&dev);
  Profiler& prof = profiler();
  const bool timed = !prof.suspended && prof.ready(dev);
  if (timed) prof.mark(0, s);
  // Large alphabets: the dense softmax pass (k_dense_soft, HBM-bound) needs
  // nothing from k_pair (latency-bound, HBM idle), so it runs on a forked
  // stream concurrently with it; the key-column patch follows both.
  OverlapStreams* ov = nullptr;
  if (!fused && dense_overlap_enabled()) {
    ov = &overlap_streams_for_current_device();
    if (!ov->init() || cudaEventRecord(ov->fork, s) != cudaSuccess ||
        cudaStreamWaitEvent(ov->side, ov->fork, 0) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
  }
  if (launch_pair(a, stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  if (timed) prof.mark(1, s);
  if (ov != nullptr) {
    if (timed) prof.mark(4, ov->side);
    const bool ok = launch_dense_soft(a, grads != nullptr, dense_exclusion_smem(a.g), ov->side) == cudaSuccess;
    if (timed) prof.mark(5, ov->side);
    // the caller's stream waits for the side stream on every path (ordering)
    if (cudaEventRecord(ov->join, ov->side) != cudaSuccess || cudaStreamWaitEvent(s, ov->join, 0) != cudaSuccess ||
        !ok)
      return DS2CTC_STATUS_EXECUTION_FAILED;
    if (launch_dense_patch(a, stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  } else if (!fused && launch_dense(a, grads != nullptr, stream) != cudaSuccess) {
    return DS2CTC_STATUS_EXECUTION_FAILED;
  }
  if (timed) prof.mark(2, s);
  if (!fused && launch_finalize(a, stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  if (timed) {
    prof.mark(3, s);
    ++prof.calls;
  }
  return DS2CTC_STATUS_SUCCESS;
}

// Descriptors + labels of the fp64 lattice paths (alignment, export) into
// the workspace head; returns the largest per-CTA shared-memory need.
ds2ctc_status stage_lattice_meta(const ViterbiLayout& lay, const int* flat_labels, const int* label_lengths,
                                 const int* input_lengths, int B, void* workspace, void* stream, size_t* smem_out) {
  const size_t meta = lay.bp;
  thread_local std::vector<unsigned char> blob;
  blob.assign(meta, 0);
  auto* desc = reinterpret_cast<ViterbiDesc*>(blob.data() + lay.desc);
  long long lab_off = 0, cell_off = 0;
  size_t smem = 0;
  for (int b = 0; b < B; ++b) {
    const int T = input_lengths[b], L = label_lengths[b];
    ViterbiDesc& d = desc[b];
    d.T = T;
    d.L = L;
    d.lab_off = static_cast<int>(lab_off);
    d.status = (T == 0 || T < min_frames(flat_labels + lab_off, L)) ? 1 : 0;  // ctc.cpp:328
    d.bp_off = cell_off;
    d.pad = 0;
    smem = std::max(smem, viterbi_smem_bytes(T, L));  // == lattice_smem_bytes
    lab_off += L;
    cell_off += static_cast<long long>(T) * (2LL * L + 1);
  }
  if (lab_off > 0) std::memcpy(blob.data() + lay.labels, flat_labels, sizeof(int) * lab_off);
  if (smem > kSmemBudget) return DS2CTC_STATUS_UNSUPPORTED;
  auto s = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev = nullptr;
  void* pinned = staging_for_current_device().acquire(meta, &ev);
  if (pinned == nullptr) return DS2CTC_STATUS_MEMOPS_FAILED;
  std::memcpy(pinned, blob.data(), meta);
  if (cudaMemcpyAsync(workspace, pinned, meta, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return DS2CTC_STATUS_MEMOPS_FAILED;
  if (cudaEventRecord(ev, s) != cudaSuccess) return DS2CTC_STATUS_MEMOPS_FAILED;
  *smem_out = smem;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status run_lattice(const float* acts, const int* flat_labels, const int* label_lengths,
                          const int* input_lengths, int A, int B, int blank, double* alpha, double* beta,
                          double* log_prob, void* workspace, size_t workspace_bytes, void* stream) {
  ds2ctc_status st = validate(label_lengths, input_lengths, A, B, blank, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  for (int b = 0; b < B; ++b)
    if (input_lengths[b] < 1) return DS2CTC_STATUS_INVALID_VALUE;  // ctc_lattice requires T >= 1 (ctc.cpp:146)
  if (B == 0) return DS2CTC_STATUS_SUCCESS;
  const ViterbiLayout lay = make_viterbi_layout(label_lengths, input_lengths, B);
  if (acts == nullptr || alpha == nullptr || beta == nullptr || log_prob == nullptr || workspace == nullptr)
    return DS2CTC_STATUS_INVALID_VALUE;
  if (workspace_bytes < lay.bp || reinterpret_cast<uintptr_t>(workspace) % kAlign != 0)
    return DS2CTC_STATUS_INVALID_VALUE;
  size_t smem = 0;
  st = stage_lattice_meta(lay, flat_labels, label_lengths, input_lengths, B, workspace, stream, &smem);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  auto* ws = static_cast<unsigned char*>(workspace);
  LatticeArgs a{};
  a.x = acts;
  a.desc = reinterpret_cast<const ViterbiDesc*>(ws + lay.desc);
  a.labels = reinterpret_cast<const int*>(ws + lay.labels);
  a.alpha = alpha;
  a.beta = beta;
  a.log_prob = log_prob;
  a.t_max = lay.t_max;
  a.B = B;
  a.A = A;
  a.blank = blank;
  if (launch_lattice(a, smem, stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status run_viterbi(const float* acts, const int* flat_labels, const int* label_lengths,
                          const int* input_lengths, int A, int B, int blank, int* alignments, int* status,
                          void* workspace, size_t workspace_bytes, void* stream) {
  ds2ctc_status st = validate(label_lengths, input_lengths, A, B, blank, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (B == 0) return DS2CTC_STATUS_SUCCESS;
  const ViterbiLayout lay = make_viterbi_layout(label_lengths, input_lengths, B);
  if (alignments == nullptr || status == nullptr || workspace == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (lay.t_max > 0 && acts == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (workspace_bytes < lay.total) return DS2CTC_STATUS_INVALID_VALUE;
  if (reinterpret_cast<uintptr_t>(workspace) % kAlign != 0) return DS2CTC_STATUS_INVALID_VALUE;
  size_t smem = 0;
  st = stage_lattice_meta(lay, flat_labels, label_lengths, input_lengths, B, workspace, stream, &smem);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  auto* ws = static_cast<unsigned char*>(workspace);
  ViterbiArgs a{};
  a.x = acts;
  a.desc = reinterpret_cast<const ViterbiDesc*>(ws + lay.desc);
  a.labels = reinterpret_cast<const int*>(ws + lay.labels);
  a.bp = ws + lay.bp;
  a.align = alignments;
  a.status = status;
  a.t_max = lay.t_max;
  a.B = B;
  a.A = A;
  a.blank = blank;
  if (launch_viterbi(a, smem, stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

// Per-thread device context of the host-buffer entry point.
// The host-buffer loss call splits the batch into up to this many contiguous
// sub-batches, each on its own stream, so that chunk c's kernels overlap chunk
// c+1's host->device copy and chunk c-1's device->host copy (PCIe, not the
// kernels, bounds this call: DESIGN.md section 8). DS2CTC_HOST_CHUNKS=1
// restores the single-stream call.
constexpr int kHostChunksMax = 8;

int host_chunks(int B, size_t bytes) {
  static const int env = [] {
    const char* v = std::getenv("DS2CTC_HOST_CHUNKS");
    return v ? std::atoi(v) : -1;
  }();
  // measured on B200: 4 chunks best at the English
  // shape (5 MB), 8 at the Mandarin one (537 MB)
  const int dflt = bytes >= (size_t{64} << 20) ? 8 : bytes >= (size_t{1} << 20) ? 4 : 1;
  int n = env > 0 ? std::min(env, kHostChunksMax) : dflt;
  return std::max(1, std::min(n, B / 4 > 0 ? B / 4 : 1));
}

bool host_direct_enabled() {
  static const bool on = [] {
    // opt-in: measured equal at the English shape (the PCIe stores stretch
    // k_pair by what they save) and 6 % slower on SortaGrad
    const char* v = std::getenv("DS2CTC_HOST_DIRECT");
    return v != nullptr && std::atoi(v) != 0;
  }();
  return on;
}

struct HostContext {
  int device = -1;
  cudaStream_t stream = nullptr;
  void* acts = nullptr;
  size_t acts_cap = 0;
  void* grads = nullptr;
  size_t grads_cap = 0;
  void* costs = nullptr;
  size_t costs_cap = 0;
  void* ws = nullptr;
  size_t ws_cap = 0;
  // extra streams of the chunked host pipeline (ds2ctc_compute_loss_host)
  cudaStream_t chunk_streams[kHostChunksMax - 1] = {};
  // end of chunk c's activation upload: chunk c + 1's upload waits for it
  cudaEvent_t uploaded[kHostChunksMax] = {};
  ~HostContext() {
    if (device < 0) return;
    cudaSetDevice(device);
    cudaFree(acts);
    cudaFree(grads);
    cudaFree(costs);
    cudaFree(ws);
    if (stream) cudaStreamDestroy(stream);
    for (cudaStream_t cs : chunk_streams)
      if (cs) cudaStreamDestroy(cs);
    for (cudaEvent_t ev : uploaded)
      if (ev) cudaEventDestroy(ev);
  }
};

bool grow(void** p, size_t* cap, size_t want) {
  if (*cap >= want) return true;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  if (want == 0) return true;
  if (cudaMalloc(p, want) != cudaSuccess) return false;
  *cap = want;
  return true;
}

// Zeroed device memory for a peer-memory collective and its CUDA IPC handle;
// freed again on any failure after the allocation.
ds2ctc_status ipc_region_alloc(size_t bytes, void** region, void* ipc_handle) {
  if (cudaMalloc(region, bytes) != cudaSuccess) return DS2CTC_STATUS_MEMOPS_FAILED;
  cudaIpcMemHandle_t h;
  ds2ctc_status st = DS2CTC_STATUS_SUCCESS;
  if (cudaMemset(*region, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    st = DS2CTC_STATUS_MEMOPS_FAILED;
  else if (cudaIpcGetMemHandle(&h, *region) != cudaSuccess)
    st = DS2CTC_STATUS_EXECUTION_FAILED;
  if (st != DS2CTC_STATUS_SUCCESS) {
    cudaFree(*region);
    *region = nullptr;
    return st;
  }
  std::memcpy(ipc_handle, &h, sizeof(h));
  return DS2CTC_STATUS_SUCCESS;
}

}  // namespace
}  // namespace ds2ctc

using namespace ds2ctc;

extern "C" {

const char* ds2ctc_status_string(ds2ctc_status status) {
  switch (status) {
    case DS2CTC_STATUS_SUCCESS: return "no error";
    case DS2CTC_STATUS_INVALID_VALUE: return "invalid value";
    case DS2CTC_STATUS_EXECUTION_FAILED: return "execution failed";
    case DS2CTC_STATUS_MEMOPS_FAILED: return "memory operation failed";
    case DS2CTC_STATUS_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

const char* ds2ctc_version(void) { return "ds2ctc 0.1.0 sm_100a"; }

// Length-split device call. A variable-length batch (SortaGrad) runs as up to
// four contiguous sub-batches, each launched with the geometry of its own
// longest label (fewer chain warps, less shared memory, more CTAs per SM for
// the short ones) on forked streams that join back into the caller's stream.
// Split only when some quarter's longest label is under 3/4 of the batch's,
// so fixed-shape batches keep the single launch. Fused path only (A <= 128):
// the sub-batch views use frame stride B.
constexpr int kDevSplitMax = 8;

struct SplitPlan {
  int n = 1;
  int b0[kDevSplitMax + 1];
  size_t lab0[kDevSplitMax];
  size_t ws_off[kDevSplitMax + 1];
};

// DS2CTC_LENGTH_SPLIT: 0 = single launch, n >= 2 = n sub-batches; default
// 8 from B = 256 up, else none. Measured SortaGrad: B = 512 (1 GPU) 230k ->
// 298k (4) / 303k (8) utt/s; B = 256 per GPU (2 GPUs) 428k -> 506k (8);
// B = 128 per GPU (4 GPUs) 780k (none) vs 773k (4) / 720k (8): one wave of
// clusters already holds the whole batch there.
int dev_split_count(int B) {
  static const int n = [] {
    const char* v = std::getenv("DS2CTC_LENGTH_SPLIT");
    const int k = v ? std::atoi(v) : -1;
    return k < 0 ? -1 : k <= 1 ? 1 : std::min(k, kDevSplitMax);
  }();
  return n > 0 ? n : (B >= 256 ? 8 : 1);
}

SplitPlan plan_split(const int* label_lengths, const int* input_lengths, int A, int B) {
  SplitPlan p;
  p.b0[0] = 0;
  p.b0[1] = B;
  p.lab0[0] = 0;
  p.ws_off[0] = 0;
  const int ns = dev_split_count(B);
  if (ns > 1 && B >= 16 * ns && A <= kFusedMaxAlphabet) {
    int lmax_all = 0, lmax_min = 1 << 30;
    for (int c = 0; c < ns; ++c) {
      int m = 0;
      for (int b = B * c / ns; b < B * (c + 1) / ns; ++b) m = std::max(m, label_lengths[b]);
      lmax_all = std::max(lmax_all, m);
      lmax_min = std::min(lmax_min, m);
    }
    if (4LL * lmax_min < 3LL * lmax_all) p.n = ns;
  }
  size_t lab = 0;
  for (int c = 0; c < p.n; ++c) {
    p.b0[c + 1] = static_cast<int>(static_cast<long long>(B) * (c + 1) / p.n);
    p.lab0[c] = lab;
    for (int b = p.b0[c]; b < p.b0[c + 1]; ++b) lab += static_cast<size_t>(label_lengths[b]);
    const size_t wsz =
        make_layout(label_lengths + p.b0[c], input_lengths + p.b0[c], A, p.b0[c + 1] - p.b0[c]).total;
    p.ws_off[c + 1] = p.ws_off[c] + (wsz + kAlign - 1) / kAlign * kAlign;
  }
  return p;
}

struct SplitStreams {
  cudaStream_t s[kDevSplitMax - 1] = {};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[kDevSplitMax - 1] = {};
  bool init() {
    if (fork) return true;
    for (auto& x : s)
      if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess) return false;
    for (auto& e : join)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return false;
    return cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess;
  }
};

ds2ctc_status run_split(const float* acts, float* grads, const int* flat_labels, const int* label_lengths,
                        const int* input_lengths, int A, int B, int blank, float* costs, void* workspace,
                        size_t workspace_bytes, bool check_ws, void* stream) {
  ds2ctc_status st = validate(label_lengths, input_lengths, A, B, blank, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS || B == 0) return st;
  const SplitPlan p = plan_split(label_lengths, input_lengths, A, B);
  if (p.n == 1)
    return run(acts, grads, flat_labels, label_lengths, input_lengths, A, B, blank, costs, workspace,
               workspace_bytes, check_ws, stream);
  if (check_ws && workspace_bytes < p.ws_off[p.n]) return DS2CTC_STATUS_INVALID_VALUE;
  if (costs == nullptr || workspace == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  thread_local std::map<int, SplitStreams> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  SplitStreams& ss = per_device[dev];
  if (!ss.init()) return DS2CTC_STATUS_EXECUTION_FAILED;
  auto s0 = static_cast<cudaStream_t>(stream);
  // stage events (ds2ctc_profile_*): k_pair = fork to join of the whole call
  Profiler& prof = profiler();
  const bool timed = prof.ready(dev);
  if (timed) prof.mark(0, s0);
  struct Suspend {
    Profiler& p;
    ~Suspend() { p.suspended = false; }
  } suspend{prof};
  prof.suspended = true;
  if (cudaEventRecord(ss.fork, s0) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  int forked = 1;  // streams ordered after the fork (s0 itself is #0)
  for (; forked < p.n; ++forked)
    if (cudaStreamWaitEvent(ss.s[forked - 1], ss.fork, 0) != cudaSuccess) break;
  // Every forked stream joins back into s0, on the error path as well, so the
  // caller's stream stays ordered after whatever the sub-batches enqueued.
  auto join = [&](ds2ctc_status result) {
    for (int c = 1; c < forked; ++c)
      if (cudaEventRecord(ss.join[c - 1], ss.s[c - 1]) != cudaSuccess ||
          cudaStreamWaitEvent(s0, ss.join[c - 1], 0) != cudaSuccess)
        result = DS2CTC_STATUS_EXECUTION_FAILED;
    return result;
  };
  if (forked < p.n) return join(DS2CTC_STATUS_EXECUTION_FAILED);
  // one staging slot for the whole call: the sub-batches' metadata blobs side by side
  size_t blob_off[kDevSplitMax + 1];
  blob_off[0] = 0;
  for (int c = 0; c < p.n; ++c)
    blob_off[c + 1] = blob_off[c] + (make_layout(label_lengths + p.b0[c], input_lengths + p.b0[c], A,
                                                 p.b0[c + 1] - p.b0[c]).meta_end + 255) / 256 * 256;
  cudaEvent_t slot_ev = nullptr;
  auto* pinned = static_cast<unsigned char*>(staging_for_current_device().acquire(blob_off[p.n], &slot_ev));
  if (pinned == nullptr) return join(DS2CTC_STATUS_MEMOPS_FAILED);
  int t_max = 0;
  for (int b = 0; b < B; ++b) t_max = std::max(t_max, input_lengths[b]);
  for (int c = 0; c < p.n; ++c) {
    const size_t col = static_cast<size_t>(p.b0[c]) * A;
    // each launch zero-fills padded rows only up to its own longest utterance:
    // the rest of this chunk's columns, up to the batch's T_max, here
    int t_c = 0;
    for (int b = p.b0[c]; b < p.b0[c + 1]; ++b) t_c = std::max(t_c, input_lengths[b]);
    const size_t pitch = static_cast<size_t>(B) * A * sizeof(float);
    if (grads && t_c < t_max &&
        cudaMemset2DAsync(grads + static_cast<size_t>(t_c) * B * A + col, pitch, 0,
                          static_cast<size_t>(p.b0[c + 1] - p.b0[c]) * A * sizeof(float), t_max - t_c,
                          c == 0 ? s0 : ss.s[c - 1]) != cudaSuccess)
      return join(DS2CTC_STATUS_EXECUTION_FAILED);
    st = run(acts + col, grads ? grads + col : nullptr, flat_labels + p.lab0[c], label_lengths + p.b0[c],
             input_lengths + p.b0[c], A, p.b0[c + 1] - p.b0[c], blank, costs + p.b0[c],
             static_cast<unsigned char*>(workspace) + p.ws_off[c], p.ws_off[c + 1] - p.ws_off[c], true,
             c == 0 ? stream : ss.s[c - 1], B, pinned + blob_off[c]);
    if (st != DS2CTC_STATUS_SUCCESS) {
      st = join(st);
      cudaEventRecord(slot_ev, s0);  // the slot is reusable once s0 passes every sub-batch's copy
      return st;
    }
  }
  st = join(DS2CTC_STATUS_SUCCESS);
  if (cudaEventRecord(slot_ev, s0) != cudaSuccess && st == DS2CTC_STATUS_SUCCESS) st = DS2CTC_STATUS_EXECUTION_FAILED;
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (timed) {
    prof.mark(1, s0);
    prof.mark(2, s0);
    prof.mark(3, s0);
    ++prof.calls;
  }
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_get_workspace_size(const int* label_lengths, const int* input_lengths, int alphabet_size,
                                        int minibatch, size_t* bytes) {
  if (bytes == nullptr || minibatch < 0 || alphabet_size < 2) return DS2CTC_STATUS_INVALID_VALUE;
  if (minibatch > 0 && (label_lengths == nullptr || input_lengths == nullptr)) return DS2CTC_STATUS_INVALID_VALUE;
  for (int b = 0; b < minibatch; ++b) {
    if (label_lengths[b] < 0 || input_lengths[b] < 0) return DS2CTC_STATUS_INVALID_VALUE;
    if (2LL * label_lengths[b] + 1 > kMaxStates) return DS2CTC_STATUS_UNSUPPORTED;
  }
  *bytes = 0;
  if (minibatch > 0) {
    const SplitPlan p = plan_split(label_lengths, input_lengths, alphabet_size, minibatch);
    *bytes = p.n == 1 ? make_layout(label_lengths, input_lengths, alphabet_size, minibatch).total : p.ws_off[p.n];
  }
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_compute_loss(const float* activations, float* gradients, const int* flat_labels,
                                  const int* label_lengths, const int* input_lengths, int alphabet_size,
                                  int minibatch, int blank_label, float* costs, void* workspace, void* stream) {
  return run_split(activations, gradients, flat_labels, label_lengths, input_lengths, alphabet_size, minibatch,
                   blank_label, costs, workspace, 0, false, stream);
}

ds2ctc_status ds2ctc_compute_loss_checked(const float* activations, float* gradients, const int* flat_labels,
                                          const int* label_lengths, const int* input_lengths, int alphabet_size,
                                          int minibatch, int blank_label, float* costs, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  return run_split(activations, gradients, flat_labels, label_lengths, input_lengths, alphabet_size, minibatch,
                   blank_label, costs, workspace, workspace_bytes, true, stream);
}

ds2ctc_status ds2ctc_viterbi_get_workspace_size(const int* label_lengths, const int* input_lengths,
                                                int alphabet_size, int minibatch, size_t* bytes) {
  if (bytes == nullptr || minibatch < 0 || alphabet_size < 2) return DS2CTC_STATUS_INVALID_VALUE;
  if (minibatch > 0 && (label_lengths == nullptr || input_lengths == nullptr)) return DS2CTC_STATUS_INVALID_VALUE;
  for (int b = 0; b < minibatch; ++b)
    if (label_lengths[b] < 0 || input_lengths[b] < 0) return DS2CTC_STATUS_INVALID_VALUE;
  *bytes = make_viterbi_layout(label_lengths, input_lengths, minibatch).total;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_viterbi_align(const float* activations, const int* flat_labels, const int* label_lengths,
                                   const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                   int* alignments, int* status, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  return run_viterbi(activations, flat_labels, label_lengths, input_lengths, alphabet_size, minibatch, blank_label,
                     alignments, status, workspace, workspace_bytes, stream);
}

ds2ctc_status ds2ctc_lattice_get_sizes(const int* label_lengths, const int* input_lengths, int minibatch,
                                       size_t* cells, size_t* workspace_bytes) {
  if (cells == nullptr || workspace_bytes == nullptr || minibatch < 0) return DS2CTC_STATUS_INVALID_VALUE;
  if (minibatch > 0 && (label_lengths == nullptr || input_lengths == nullptr)) return DS2CTC_STATUS_INVALID_VALUE;
  size_t n = 0;
  for (int b = 0; b < minibatch; ++b) {
    if (label_lengths[b] < 0 || input_lengths[b] < 0) return DS2CTC_STATUS_INVALID_VALUE;
    n += static_cast<size_t>(input_lengths[b]) * (2 * static_cast<size_t>(label_lengths[b]) + 1);
  }
  *cells = n;
  *workspace_bytes = make_viterbi_layout(label_lengths, input_lengths, minibatch).bp;  // metadata only
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_ctc_lattice(const float* activations, const int* flat_labels, const int* label_lengths,
                                 const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                 double* alpha, double* beta, double* log_prob, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  return run_lattice(activations, flat_labels, label_lengths, input_lengths, alphabet_size, minibatch, blank_label,
                     alpha, beta, log_prob, workspace, workspace_bytes, stream);
}

ds2ctc_status ds2ctc_mailbox_alloc(int world, void** mailbox, void* ipc_handle) {
  if (mailbox == nullptr || ipc_handle == nullptr || world < 1 || world > kMaxPeers) return DS2CTC_STATUS_INVALID_VALUE;
  return ipc_region_alloc(mailbox_bytes(world), mailbox, ipc_handle);
}

ds2ctc_status ds2ctc_mailbox_open(const void* ipc_handle, void** peer_mailbox) {
  if (ipc_handle == nullptr || peer_mailbox == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  if (cudaIpcOpenMemHandle(peer_mailbox, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_mailbox_close(void* peer_mailbox, int own) {
  if (peer_mailbox == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  const cudaError_t e = own ? cudaFree(peer_mailbox) : cudaIpcCloseMemHandle(peer_mailbox);
  return e == cudaSuccess ? DS2CTC_STATUS_SUCCESS : DS2CTC_STATUS_EXECUTION_FAILED;
}

ds2ctc_status ds2ctc_exchange_size(size_t n, size_t* bytes) {
  if (bytes == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  *bytes = vec_exchange_bytes(static_cast<long long>(n));
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_exchange_alloc(size_t bytes, void** region, void* ipc_handle) {
  if (region == nullptr || ipc_handle == nullptr || bytes == 0) return DS2CTC_STATUS_INVALID_VALUE;
  return ipc_region_alloc(bytes, region, ipc_handle);
}

ds2ctc_status ds2ctc_vec_allreduce(float* data, size_t n, void* const* peer_regions, int rank, int world,
                                   unsigned long long seq, void* stream) {
  if ((n > 0 && data == nullptr) || peer_regions == nullptr || world < 1 || world > kMaxPeers || rank < 0 ||
      rank >= world || seq == 0)
    return DS2CTC_STATUS_INVALID_VALUE;
  PeerMailboxes pr{};
  for (int r = 0; r < world; ++r) {
    if (peer_regions[r] == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
    pr.peer[r] = peer_regions[r];
  }
  pr.rank = rank;
  pr.world = world;
  if (launch_vec_allreduce(data, static_cast<long long>(n), pr, seq, stream) != cudaSuccess)
    return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_loss_sum_allreduce(const float* costs, int minibatch, double* out2, void* const* peer_mailboxes,
                                        int rank, int world, unsigned long long seq, void* stream) {
  if (out2 == nullptr || minibatch < 0 || (minibatch > 0 && costs == nullptr) || peer_mailboxes == nullptr ||
      world < 1 || world > kMaxPeers || rank < 0 || rank >= world || seq == 0)
    return DS2CTC_STATUS_INVALID_VALUE;
  PeerMailboxes mb{};
  for (int r = 0; r < world; ++r) {
    if (peer_mailboxes[r] == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
    mb.peer[r] = peer_mailboxes[r];
  }
  mb.rank = rank;
  mb.world = world;
  if (launch_loss_allreduce(costs, minibatch, out2, mb, seq, stream) != cudaSuccess)
    return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_reduce_fault(unsigned long long* seq) {
  if (seq == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (read_reduce_fault(seq) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_loss_sum(const float* costs, int minibatch, double* out2, void* stream) {
  if (minibatch < 0 || out2 == nullptr || (minibatch > 0 && costs == nullptr)) return DS2CTC_STATUS_INVALID_VALUE;
  if (launch_loss_sum(costs, minibatch, out2, stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_fc_backward_workspace_size(int rows, int out_dim, int in_dim, size_t* bytes) {
  if (bytes == nullptr || rows < 0 || out_dim < 1 || in_dim < 1) return DS2CTC_STATUS_INVALID_VALUE;
  *bytes = fc_backward_workspace(rows, out_dim, in_dim);
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_fc_backward(const float* dlogits, const float* x, const float* w, float* dw, float* db, float* dx,
                                 int rows, int out_dim, int in_dim, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  if (rows < 0 || out_dim < 1 || in_dim < 1) return DS2CTC_STATUS_INVALID_VALUE;
  if (rows == 0) return DS2CTC_STATUS_SUCCESS;
  if (dlogits == nullptr || (dw != nullptr && x == nullptr) || (dx != nullptr && w == nullptr))
    return DS2CTC_STATUS_INVALID_VALUE;
  // TMA: 16-byte aligned bases and row pitches (in_dim % 4 == 0); the gradient
  // rows are re-pitched into the workspace when out_dim % 4 != 0
  if (in_dim % 4 != 0) return DS2CTC_STATUS_UNSUPPORTED;
  for (const void* p : {static_cast<const void*>(dlogits), static_cast<const void*>(x), static_cast<const void*>(w),
                        static_cast<const void*>(dx)})
    if (p != nullptr && reinterpret_cast<uintptr_t>(p) % 16 != 0) return DS2CTC_STATUS_INVALID_VALUE;
  const size_t need = fc_backward_workspace(rows, out_dim, in_dim);
  if (workspace_bytes < need || (need > 0 && (workspace == nullptr || reinterpret_cast<uintptr_t>(workspace) % 256)))
    return DS2CTC_STATUS_INVALID_VALUE;
  if (fc_backward(dlogits, x, w, dw, db, dx, rows, out_dim, in_dim, workspace, sm_count(), stream) != cudaSuccess)
    return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_profile_enable(int slots) {
  if (slots < 0) return DS2CTC_STATUS_INVALID_VALUE;
  Profiler& p = profiler();
  p.reset();
  p.slots = slots;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_profile_read(int call_index, float* ms) {
  Profiler& p = profiler();
  if (ms == nullptr || call_index < 0 || call_index >= p.calls) return DS2CTC_STATUS_INVALID_VALUE;
  cudaEvent_t* e = p.ev.data() + 6 * call_index;
  if (cudaEventSynchronize(e[3]) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  const bool side = p.side[call_index] != 0;
  if (cudaEventElapsedTime(&ms[0], e[0], e[1]) != cudaSuccess ||
      cudaEventElapsedTime(&ms[1], side ? e[4] : e[1], side ? e[5] : e[2]) != cudaSuccess ||
      cudaEventElapsedTime(&ms[2], e[2], e[3]) != cudaSuccess ||
      cudaEventElapsedTime(&ms[3], e[0], e[3]) != cudaSuccess)
    return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_debug_watchdog(unsigned long long* out4) {
  if (out4 == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (cudaDeviceSynchronize() != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  if (read_watchdog(out4) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_compute_loss_host(const float* activations, float* gradients, const int* flat_labels,
                                       const int* label_lengths, const int* input_lengths, int alphabet_size,
                                       int minibatch, int blank_label, float* costs, int device) {
  ds2ctc_status st = validate(label_lengths, input_lengths, alphabet_size, minibatch, blank_label, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (minibatch == 0) return DS2CTC_STATUS_SUCCESS;
  if (costs == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  thread_local std::map<int, HostContext> contexts;
  if (cudaSetDevice(device) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  HostContext& ctx = contexts[device];
  if (ctx.device < 0) {
    ctx.device = device;
    if (cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
  }
  const int A = alphabet_size, B = minibatch;
  const Layout lay = make_layout(label_lengths, input_lengths, A, B);
  const size_t elems = static_cast<size_t>(lay.t_max) * B * A;
  if (elems > 0 && activations == nullptr) return DS2CTC_STATUS_INVALID_VALUE;

  // Chunk c = utterances [b0[c], b0[c+1]): its activations land compactly as
  // [T_c][B_c][A] (T_c = the chunk's longest utterance) at a 256-byte aligned
  // offset, with a workspace of its own.
  const int nc = host_chunks(B, elems * sizeof(float));
  // Direct mode (DS2CTC_HOST_DIRECT=1): a page-locked (UVA-mapped) gradient buffer on the fused path
  // (A <= 128) is written by k_pair itself over PCIe as the rows are produced,
  // so no device->host gradient copy trails the kernels. The activations then
  // land in a full [T][B][A] device buffer (chunk c's columns), and each chunk
  // runs as a sub-batch view with frame stride B.
  float* g_direct = nullptr;
  if (gradients && alphabet_size <= kFusedMaxAlphabet && host_direct_enabled()) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, gradients) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer != nullptr)
      g_direct = static_cast<float*>(pa.devicePointer);
    else
      cudaGetLastError();
  }
  const bool direct = g_direct != nullptr;
  int b0[kHostChunksMax + 1];
  int t_c[kHostChunksMax];
  size_t lab0[kHostChunksMax], x_off[kHostChunksMax], ws_off[kHostChunksMax + 1];
  size_t x_total = 0, lab = 0;
  ws_off[0] = 0;
  for (int c = 0; c <= nc; ++c) b0[c] = static_cast<int>(static_cast<long long>(B) * c / nc);
  for (int c = 0; c < nc; ++c) {
    const int bc = b0[c + 1] - b0[c];
    t_c[c] = 0;
    lab0[c] = lab;
    for (int b = b0[c]; b < b0[c + 1]; ++b) {
      t_c[c] = std::max(t_c[c], input_lengths[b]);
      lab += static_cast<size_t>(label_lengths[b]);
    }
    if (direct) {
      x_off[c] = static_cast<size_t>(b0[c]) * A * sizeof(float);
      x_total = elems * sizeof(float);
    } else {
      x_off[c] = x_total;
      x_total += (static_cast<size_t>(t_c[c]) * bc * A * sizeof(float) + kAlign - 1) / kAlign * kAlign;
    }
    const size_t wsz = nc == 1 ? lay.total : make_layout(label_lengths + b0[c], input_lengths + b0[c], A, bc).total;
    ws_off[c + 1] = ws_off[c] + (wsz + kAlign - 1) / kAlign * kAlign;
  }
  if (!grow(&ctx.acts, &ctx.acts_cap, x_total) ||
      !grow(&ctx.grads, &ctx.grads_cap, gradients && !direct ? x_total : 0) ||
      !grow(&ctx.costs, &ctx.costs_cap, B * sizeof(float)) || !grow(&ctx.ws, &ctx.ws_cap, ws_off[nc]))
    return DS2CTC_STATUS_MEMOPS_FAILED;
  for (int c = 1; c < nc; ++c)
    if (!ctx.chunk_streams[c - 1] &&
        cudaStreamCreateWithFlags(&ctx.chunk_streams[c - 1], cudaStreamNonBlocking) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
  for (int c = 0; c + 1 < nc; ++c)
    if (!ctx.uploaded[c] && cudaEventCreateWithFlags(&ctx.uploaded[c], cudaEventDisableTiming) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
  // Uploads in chunk order, one at a time (DS2CTC_HOST_SERIAL_UPLOAD=0: all at
  // once). Issued concurrently, the chunks' copies share PCIe and all land at
  // the end of the whole upload, so every chunk's kernels start late; one at a
  // time, chunk 0's k_pair starts after a quarter of it and only the last
  // chunk's kernels trail the upload.
  static const bool serial_upload = [] {
    const char* v = std::getenv("DS2CTC_HOST_SERIAL_UPLOAD");
    return v == nullptr || std::atoi(v) != 0;
  }();

  const size_t row = static_cast<size_t>(B) * A * sizeof(float);
  // The contract is synchronous: on an error after some chunk was enqueued,
  // drain every chunk stream before returning, so no queued copy touches the
  // caller's host buffers after the call.
  auto drain = [&](ds2ctc_status result) {
    for (int c = 0; c < nc; ++c)
      if (cudaStreamSynchronize(c == 0 ? ctx.stream : ctx.chunk_streams[c - 1]) != cudaSuccess)
        result = result == DS2CTC_STATUS_SUCCESS ? DS2CTC_STATUS_EXECUTION_FAILED : result;
    return result;
  };
  // Two passes over the chunks: every upload and kernel launch first, then
  // the downloads. The host's enqueue work per chunk (metadata, copies,
  // launch: ~20-30 us) then stays ahead of the serialised uploads, so the
  // last chunk's k_pair is not waiting for the host to enqueue the earlier
  // chunks' downloads (DS2CTC_HOST_TWO_PASS=0: one pass).
  static const bool two_pass = [] {
    const char* v = std::getenv("DS2CTC_HOST_TWO_PASS");
    return v == nullptr || std::atoi(v) != 0;
  }();
  auto chunk_stream = [&](int c) { return c == 0 ? ctx.stream : ctx.chunk_streams[c - 1]; };
  auto chunk_width = [&](int c) { return static_cast<size_t>(b0[c + 1] - b0[c]) * A * sizeof(float); };
  auto chunk_grads = [&](int c) -> unsigned char* {
    return !gradients ? nullptr
           : direct   ? reinterpret_cast<unsigned char*>(g_direct) + x_off[c]
                      : static_cast<unsigned char*>(ctx.grads) + x_off[c];
  };
  auto launch = [&](int c) -> ds2ctc_status {
    cudaStream_t sc = chunk_stream(c);
    const int bc = b0[c + 1] - b0[c];
    const size_t w = chunk_width(c);
    auto* xd = static_cast<unsigned char*>(ctx.acts) + x_off[c];
    const size_t xpitch = direct ? row : w;
    const auto* xh = reinterpret_cast<const unsigned char*>(activations) + static_cast<size_t>(b0[c]) * A * sizeof(float);
    if (serial_upload && c > 0 && cudaStreamWaitEvent(sc, ctx.uploaded[c - 1], 0) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
    if (t_c[c] > 0 && w > 0 &&
        cudaMemcpy2DAsync(xd, xpitch, xh, row, w, t_c[c], cudaMemcpyHostToDevice, sc) != cudaSuccess)
      return DS2CTC_STATUS_MEMOPS_FAILED;
    if (serial_upload && c + 1 < nc && cudaEventRecord(ctx.uploaded[c], sc) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
    float* cd = static_cast<float*>(ctx.costs) + b0[c];
    return run(reinterpret_cast<const float*>(xd), reinterpret_cast<float*>(chunk_grads(c)), flat_labels + lab0[c],
               label_lengths + b0[c], input_lengths + b0[c], A, bc, blank_label, cd,
               static_cast<unsigned char*>(ctx.ws) + ws_off[c], ws_off[c + 1] - ws_off[c], true, sc, direct ? B : 0);
  };
  auto download = [&](int c) -> ds2ctc_status {
    cudaStream_t sc = chunk_stream(c);
    const int bc = b0[c + 1] - b0[c];
    const size_t w = chunk_width(c);
    if (gradients && t_c[c] > 0 && w > 0) {
      auto* gh = reinterpret_cast<unsigned char*>(gradients) + static_cast<size_t>(b0[c]) * A * sizeof(float);
      if (!direct && cudaMemcpy2DAsync(gh, row, chunk_grads(c), w, w, t_c[c], cudaMemcpyDeviceToHost, sc) != cudaSuccess)
        return DS2CTC_STATUS_MEMOPS_FAILED;
      // frames past this chunk's longest utterance: zero rows (the contract), on the host
      for (int t = t_c[c]; t < lay.t_max; ++t) std::memset(gh + static_cast<size_t>(t) * row, 0, w);
    }
    float* cd = static_cast<float*>(ctx.costs) + b0[c];
    if (bc > 0 && cudaMemcpyAsync(costs + b0[c], cd, bc * sizeof(float), cudaMemcpyDeviceToHost, sc) != cudaSuccess)
      return DS2CTC_STATUS_MEMOPS_FAILED;
    return DS2CTC_STATUS_SUCCESS;
  };
  for (int c = 0; c < nc; ++c) {
    st = launch(c);
    if (st == DS2CTC_STATUS_SUCCESS && !two_pass) st = download(c);
    if (st != DS2CTC_STATUS_SUCCESS) return drain(st);
  }
  if (two_pass)
    for (int c = 0; c < nc; ++c)
      if ((st = download(c)) != DS2CTC_STATUS_SUCCESS) return drain(st);
  return drain(DS2CTC_STATUS_SUCCESS);
}

// Host-buffer forms of the alignment and lattice export (the C++ shim's
// per-utterance viterbi_align / ctc_lattice): copies through the per-thread
// device context, synchronous.
ds2ctc_status ds2ctc_viterbi_align_host(const float* activations, const int* flat_labels, const int* label_lengths,
                                        const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                        int* alignments, int* status, int device) {
  ds2ctc_status st = validate(label_lengths, input_lengths, alphabet_size, minibatch, blank_label, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (minibatch == 0) return DS2CTC_STATUS_SUCCESS;
  if (alignments == nullptr || status == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  thread_local std::map<int, HostContext> contexts;
  if (cudaSetDevice(device) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  HostContext& ctx = contexts[device];
  if (ctx.device < 0) {
    ctx.device = device;
    if (cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
  }
  const ViterbiLayout lay = make_viterbi_layout(label_lengths, input_lengths, minibatch);
  const size_t elems = static_cast<size_t>(lay.t_max) * minibatch * alphabet_size;
  const size_t out_bytes = sizeof(int) * (static_cast<size_t>(lay.t_max) * minibatch + minibatch);
  if (elems > 0 && activations == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  if (!grow(&ctx.acts, &ctx.acts_cap, elems * sizeof(float)) || !grow(&ctx.grads, &ctx.grads_cap, out_bytes) ||
      !grow(&ctx.ws, &ctx.ws_cap, lay.total))
    return DS2CTC_STATUS_MEMOPS_FAILED;
  if (elems > 0 &&
      cudaMemcpyAsync(ctx.acts, activations, elems * sizeof(float), cudaMemcpyHostToDevice, ctx.stream) != cudaSuccess)
    return DS2CTC_STATUS_MEMOPS_FAILED;
  int* d_align = static_cast<int*>(ctx.grads);
  int* d_status = d_align + static_cast<size_t>(lay.t_max) * minibatch;
  st = run_viterbi(static_cast<const float*>(ctx.acts), flat_labels, label_lengths, input_lengths, alphabet_size,
                   minibatch, blank_label, d_align, d_status, ctx.ws, ctx.ws_cap, ctx.stream);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (cudaMemcpyAsync(alignments, d_align, sizeof(int) * static_cast<size_t>(lay.t_max) * minibatch,
                      cudaMemcpyDeviceToHost, ctx.stream) != cudaSuccess ||
      cudaMemcpyAsync(status, d_status, sizeof(int) * minibatch, cudaMemcpyDeviceToHost, ctx.stream) != cudaSuccess)
    return DS2CTC_STATUS_MEMOPS_FAILED;
  if (cudaStreamSynchronize(ctx.stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_ctc_lattice_host(const float* activations, const int* flat_labels, const int* label_lengths,
                                      const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                      double* alpha, double* beta, double* log_prob, int device) {
  ds2ctc_status st = validate(label_lengths, input_lengths, alphabet_size, minibatch, blank_label, flat_labels);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (minibatch == 0) return DS2CTC_STATUS_SUCCESS;
  if (alpha == nullptr || beta == nullptr || log_prob == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  thread_local std::map<int, HostContext> contexts;
  if (cudaSetDevice(device) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  HostContext& ctx = contexts[device];
  if (ctx.device < 0) {
    ctx.device = device;
    if (cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking) != cudaSuccess)
      return DS2CTC_STATUS_EXECUTION_FAILED;
  }
  const ViterbiLayout lay = make_viterbi_layout(label_lengths, input_lengths, minibatch);
  size_t cells = 0;
  for (int b = 0; b < minibatch; ++b)
    cells += static_cast<size_t>(input_lengths[b]) * (2 * static_cast<size_t>(label_lengths[b]) + 1);
  const size_t elems = static_cast<size_t>(lay.t_max) * minibatch * alphabet_size;
  if (elems > 0 && activations == nullptr) return DS2CTC_STATUS_INVALID_VALUE;
  const size_t out_bytes = sizeof(double) * (2 * cells + minibatch);
  if (!grow(&ctx.acts, &ctx.acts_cap, elems * sizeof(float)) || !grow(&ctx.grads, &ctx.grads_cap, out_bytes) ||
      !grow(&ctx.ws, &ctx.ws_cap, lay.bp))
    return DS2CTC_STATUS_MEMOPS_FAILED;
  if (elems > 0 &&
      cudaMemcpyAsync(ctx.acts, activations, elems * sizeof(float), cudaMemcpyHostToDevice, ctx.stream) != cudaSuccess)
    return DS2CTC_STATUS_MEMOPS_FAILED;
  double* d_alpha = static_cast<double*>(ctx.grads);
  double* d_beta = d_alpha + cells;
  double* d_lp = d_beta + cells;
  st = run_lattice(static_cast<const float*>(ctx.acts), flat_labels, label_lengths, input_lengths, alphabet_size,
                   minibatch, blank_label, d_alpha, d_beta, d_lp, ctx.ws, ctx.ws_cap, ctx.stream);
  if (st != DS2CTC_STATUS_SUCCESS) return st;
  if (cudaMemcpyAsync(alpha, d_alpha, sizeof(double) * cells, cudaMemcpyDeviceToHost, ctx.stream) != cudaSuccess ||
      cudaMemcpyAsync(beta, d_beta, sizeof(double) * cells, cudaMemcpyDeviceToHost, ctx.stream) != cudaSuccess ||
      cudaMemcpyAsync(log_prob, d_lp, sizeof(double) * minibatch, cudaMemcpyDeviceToHost, ctx.stream) != cudaSuccess)
    return DS2CTC_STATUS_MEMOPS_FAILED;
  if (cudaStreamSynchronize(ctx.stream) != cudaSuccess) return DS2CTC_STATUS_EXECUTION_FAILED;
  return DS2CTC_STATUS_SUCCESS;
}

}  // extern "C"
