// ds2ctc.hpp -- header-only C++ shim over the C-ABI with the reference's
// own CTC signature, so reference-style callers and tests can switch
// implementations by name:
//
//   asr::ctc::CtcResult asr::ctc::ctc_loss_reference(const Matrix& frame_logits,
//                                                    const std::vector<int>& label, int blank);
//   (/root/reference/proj/include/asr/ctc.hpp:84-87)
//
//   template <class M> ds2ctc::CtcResult<M> ds2ctc::ctc_loss_gpu(const M& frame_logits,
//                                                            const std::vector<int>& label, int blank);
//
// M is any row-major matrix type with rows(), cols(), operator()(r, c) and a
// (rows, cols) constructor -- asr::Matrix qualifies unchanged. The result
// mirrors asr::ctc::CtcResult (ctc.hpp:62-66): feasible, loss = -log p,
// logit_grad T x A (empty when infeasible). Computation runs on `device`
// through ds2ctc_compute_loss_host (fp32 in/out, fp64 lattice carry).
//
// ctc_loss_batch_gpu is the batched form the trainer loop
// (proj/src/trainer.cpp:155-171) maps onto: one call for the whole local
// minibatch instead of one ctc_loss_reference per utterance, with the
// trainer's convention already applied (infeasible -> zero gradient).
#ifndef DS2CTC_HPP
#define DS2CTC_HPP

#include <algorithm>
#include <cmath>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ds2ctc.h"

namespace ds2ctc {

template <class M>
struct CtcResult {
  bool feasible = false;
  double loss = std::numeric_limits<double>::infinity();
  M logit_grad;  // T x A; empty when infeasible

  // Converts to any result type with the reference's fields, so a caller
  // that spells the type out keeps compiling after the one-identifier switch:
  //   asr::ctc::CtcResult res = ds2ctc::ctc_loss_gpu(logits, label, blank);
  // (asr::ctc::CtcResult, ctc.hpp:62-66: feasible, loss, logit_grad)
  template <class R, class = decltype(std::declval<R&>().feasible = true, std::declval<R&>().loss = 0.0,
                                      std::declval<R&>().logit_grad = std::declval<const M&>())>
  operator R() const {
    R r;
    r.feasible = feasible;
    r.loss = static_cast<decltype(r.loss)>(loss);
    r.logit_grad = logit_grad;
    return r;
  }
};

inline void check(ds2ctc_status st, const char* where) {
  if (st != DS2CTC_STATUS_SUCCESS)
    throw std::runtime_error(std::string("ds2ctc: ") + where + ": " + ds2ctc_status_string(st));
}

template <class M>
CtcResult<M> ctc_loss_gpu(const M& frame_logits, const std::vector<int>& label, int blank, int device = 0) {
  const int T = frame_logits.rows();
  const int A = frame_logits.cols();
  std::vector<float> x(static_cast<size_t>(T) * A), g(x.size());
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < A; ++k) x[static_cast<size_t>(t) * A + k] = static_cast<float>(frame_logits(t, k));
  const int L = static_cast<int>(label.size());
  float cost = 0.f;
  check(ds2ctc_compute_loss_host(x.data(), g.data(), label.data(), &L, &T, A, 1, blank, &cost, device),
        "ctc_loss_gpu");
  CtcResult<M> res;
  if (std::isinf(cost) && cost > 0) return res;  // infeasible (ctc.cpp:173,189-193); NaN stays feasible
  res.feasible = true;
  res.loss = cost;
  res.logit_grad = M(T, A);
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < A; ++k) res.logit_grad(t, k) = g[static_cast<size_t>(t) * A + k];
  return res;
}

// Batched: logits[i] is T_i x A. Returns per-utterance costs (+inf when
// infeasible) and fills dlogits[i] (T_i x A, zero when infeasible).
template <class M>
std::vector<double> ctc_loss_batch_gpu(const std::vector<M>& logits, const std::vector<std::vector<int>>& labels,
                                       int blank, std::vector<M>* dlogits, int device = 0) {
  const int B = static_cast<int>(logits.size());
  if (B == 0) return {};
  const int A = logits[0].cols();
  std::vector<int> il(B), ll(B), flat;
  int t_max = 0;
  for (int b = 0; b < B; ++b) {
    il[b] = logits[b].rows();
    ll[b] = static_cast<int>(labels[b].size());
    t_max = std::max(t_max, il[b]);
    flat.insert(flat.end(), labels[b].begin(), labels[b].end());
  }
  std::vector<float> x(static_cast<size_t>(t_max) * B * A, 0.f), g(dlogits ? x.size() : 0);
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < il[b]; ++t)
      for (int k = 0; k < A; ++k) x[(static_cast<size_t>(t) * B + b) * A + k] = static_cast<float>(logits[b](t, k));
  std::vector<float> costs(B);
  check(ds2ctc_compute_loss_host(x.data(), dlogits ? g.data() : nullptr, flat.data(), ll.data(), il.data(), A, B,
                                 blank, costs.data(), device),
        "ctc_loss_batch_gpu");
  if (dlogits) {
    dlogits->clear();
    for (int b = 0; b < B; ++b) {
      M d(il[b], A);
      for (int t = 0; t < il[b]; ++t)
        for (int k = 0; k < A; ++k) d(t, k) = g[(static_cast<size_t>(t) * B + b) * A + k];
      dlogits->push_back(std::move(d));
    }
  }
  return std::vector<double>(costs.begin(), costs.end());
}

// std::vector<int> asr::ctc::viterbi_align(const Matrix& frame_logprobs,
//                                          const std::vector<int>& label, int blank)
// (ctc.hpp:97-101, ctc.cpp:327-370): frame symbols of the best alignment;
// throws where the reference throws (label infeasible for T, or no path).
template <class M>
std::vector<int> viterbi_align_gpu(const M& frame_logits, const std::vector<int>& label, int blank, int device = 0) {
  const int T = frame_logits.rows();
  const int A = frame_logits.cols();
  std::vector<float> x(static_cast<size_t>(T) * A);
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < A; ++k) x[static_cast<size_t>(t) * A + k] = static_cast<float>(frame_logits(t, k));
  const int L = static_cast<int>(label.size());
  std::vector<int> out(static_cast<size_t>(T > 0 ? T : 1));
  int status = 1;
  check(ds2ctc_viterbi_align_host(x.data(), label.data(), &L, &T, A, 1, blank, out.data(), &status, device),
        "viterbi_align_gpu");
  if (status != 0) throw std::runtime_error("ds2ctc: viterbi_align: label infeasible for frame count or no path");
  out.resize(static_cast<size_t>(T));
  return out;
}

// asr::ctc::CtcLattice (ctc.hpp:55-60) and ctc_lattice (ctc.cpp:145-169).
template <class M>
struct CtcLattice {
  std::vector<int> augmented_label;
  M alpha;  // (2L+1) x T
  M beta;   // (2L+1) x T, emission-exclusive
  double log_prob = -std::numeric_limits<double>::infinity();

  // To asr::ctc::CtcLattice (ctc.hpp:55-60) or any type with these fields.
  template <class R, class = decltype(std::declval<R&>().augmented_label = std::vector<int>(),
                                      std::declval<R&>().alpha = std::declval<const M&>(),
                                      std::declval<R&>().log_prob = 0.0)>
  operator R() const {
    R r;
    r.augmented_label = augmented_label;
    r.alpha = alpha;
    r.beta = beta;
    r.log_prob = static_cast<decltype(r.log_prob)>(log_prob);
    return r;
  }
};

template <class M>
CtcLattice<M> ctc_lattice_gpu(const M& frame_logits, const std::vector<int>& label, int blank, int device = 0) {
  const int T = frame_logits.rows();
  const int A = frame_logits.cols();
  if (T < 1) throw std::runtime_error("ds2ctc: ctc_lattice: need at least one frame");
  std::vector<float> x(static_cast<size_t>(T) * A);
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < A; ++k) x[static_cast<size_t>(t) * A + k] = static_cast<float>(frame_logits(t, k));
  const int L = static_cast<int>(label.size());
  const int S = 2 * L + 1;
  std::vector<double> a(static_cast<size_t>(S) * T), b(a.size());
  CtcLattice<M> lat;
  check(ds2ctc_ctc_lattice_host(x.data(), label.data(), &L, &T, A, 1, blank, a.data(), b.data(), &lat.log_prob,
                                device),
        "ctc_lattice_gpu");
  lat.augmented_label.push_back(blank);
  for (int c : label) {
    lat.augmented_label.push_back(c);
    lat.augmented_label.push_back(blank);
  }
  lat.alpha = M(S, T);
  lat.beta = M(S, T);
  for (int s = 0; s < S; ++s)
    for (int t = 0; t < T; ++t) {
      lat.alpha(s, t) = a[static_cast<size_t>(s) * T + t];
      lat.beta(s, t) = b[static_cast<size_t>(s) * T + t];
    }
  return lat;
}

// dump_lattice_tsv (ctc.cpp:372-383, declared ctc.hpp:104-105): for "alpha"
// then "beta", a header line "# <name> (<rows> x <cols>)" and one line per
// augmented position -- its symbol, then the row's values tab-separated, in
// the stream's current number format. Takes ds2ctc::CtcLattice or any lattice
// type with the same fields (asr::ctc::CtcLattice), so the debug printer
// works on what ctc_lattice_gpu returns without the reference library.
template <class Lattice>
void dump_lattice_tsv(const Lattice& lat, std::ostream& os) {
  auto one = [&](const char* name, const auto& m) {
    os << "# " << name << " (" << m.rows() << " x " << m.cols() << ")\n";
    for (int s = 0; s < m.rows(); ++s) {
      os << lat.augmented_label[static_cast<size_t>(s)];
      for (int t = 0; t < m.cols(); ++t) os << '\t' << m(s, t);
      os << '\n';
    }
  };
  one("alpha", lat.alpha);
  one("beta", lat.beta);
}

}  // namespace ds2ctc

#endif  // DS2CTC_HPP
