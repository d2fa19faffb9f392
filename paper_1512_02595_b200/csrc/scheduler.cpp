// scheduler.cpp -- H1, the host scheduler of the data-parallel CTC step.
//
// Reference: asr::trainer::train_epoch orders utterances with SortaGrad
// (sortagrad_order, proj/src/trainer.cpp:58-91) and hands each rank a
// contiguous minibatch_size slice of every global minibatch
// (trainer.cpp:140-143). That slicing of a length-sorted batch gives rank 0
// the shortest and rank N-1 the longest utterances, so the
// B200 scheduler keeps SortaGrad for batch COMPOSITION and re-deals each
// batch across GPUs longest-processing-time first. Per-utterance results do
// not depend on the deal, so parity is unaffected.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "ds2ctc.h"

namespace {

// asr::Rng, proj/include/asr/common.hpp:92-127 (SplitMix64 + Fisher-Yates).
class Rng {
 public:
  explicit Rng(uint64_t seed) : state_(seed) {}
  uint64_t next_u64() {
    uint64_t z = (state_ += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t below(uint64_t n) { return next_u64() % n; }
  template <typename T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
  }

 private:
  uint64_t state_;
};

}  // namespace

extern "C" {

ds2ctc_status ds2ctc_sortagrad_order(const int* lengths, int n, int global_batch, int epoch, uint64_t seed,
                                     int sortagrad_on, int64_t* out_order) {
  if (n < 0 || global_batch < 1 || (n > 0 && (lengths == nullptr || out_order == nullptr)))
    return DS2CTC_STATUS_INVALID_VALUE;
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  Rng rng(seed * 0x9e3779b9ULL + static_cast<uint64_t>(epoch) + 1);
  if (!sortagrad_on) {
    rng.shuffle(idx);
    std::copy(idx.begin(), idx.end(), out_order);
    return DS2CTC_STATUS_SUCCESS;
  }
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return lengths[a] < lengths[b]; });
  if (epoch == 0) {
    std::copy(idx.begin(), idx.end(), out_order);
    return DS2CTC_STATUS_SUCCESS;
  }
  const size_t batches = (static_cast<size_t>(n) + global_batch - 1) / global_batch;
  std::vector<size_t> order(batches);
  std::iota(order.begin(), order.end(), 0);
  rng.shuffle(order);
  size_t k = 0;
  for (size_t bi : order) {
    const size_t begin = bi * global_batch;
    const size_t end = std::min(static_cast<size_t>(n), begin + global_batch);
    for (size_t i = begin; i < end; ++i) out_order[k++] = idx[i];
  }
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_rank_slice(int batch_n, int minibatch_size, int rank, int* begin, int* end) {
  if (batch_n < 0 || minibatch_size < 1 || rank < 0 || begin == nullptr || end == nullptr)
    return DS2CTC_STATUS_INVALID_VALUE;
  const long long b = std::min<long long>(batch_n, static_cast<long long>(rank) * minibatch_size);
  const long long e = std::min<long long>(batch_n, (static_cast<long long>(rank) + 1) * minibatch_size);
  *begin = static_cast<int>(b);
  *end = static_cast<int>(e);
  return DS2CTC_STATUS_SUCCESS;
}

ds2ctc_status ds2ctc_shard_lpt(const int* input_lengths, const int* label_lengths, int n, int alphabet_size,
                               int world, int* out_rank, double* out_load) {
  if (n < 0 || world < 1 || alphabet_size < 1 ||
      (n > 0 && (input_lengths == nullptr || label_lengths == nullptr || out_rank == nullptr)))
    return DS2CTC_STATUS_INVALID_VALUE;
  // Estimated work per utterance: T_b frames of the serial alpha||beta chain
  // (latency-bound, A=29) and T_b * A * 8 bytes of HBM traffic (A=6000);
  // both scale with T_b within a batch (A is shared), so LPT on T_b, with
  // the lattice height 2L+1 as the tie-break.
  std::vector<double> cost(n);
  for (int i = 0; i < n; ++i) cost[i] = static_cast<double>(input_lengths[i]) * (1.0 + alphabet_size / 1024.0);
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    return label_lengths[a] > label_lengths[b];
  });
  std::vector<double> load(world, 0.0);
  std::vector<int> count(world, 0);
  for (int i : idx) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best] || (load[r] == load[best] && count[r] < count[best])) best = r;
    out_rank[i] = best;
    load[best] += cost[i];
    ++count[best];
  }
  if (out_load != nullptr) std::copy(load.begin(), load.end(), out_load);
  return DS2CTC_STATUS_SUCCESS;
}

}  // extern "C"
