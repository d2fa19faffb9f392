// C++ caller of the drop-in shim (include/ds2ctc.hpp): the reference-style
// per-utterance call ctc_loss_gpu(Matrix, label, blank) and the batched form,
// checked against the fp64 oracle restatement (oracle/ctc_oracle.h, the
// checker). Built by tests/cpp/Makefile; run by tests/test_gpu_cpp.py on a GPU.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ctc_oracle.h"
#include "ds2ctc.hpp"

namespace {

// Minimal row-major matrix with asr::Matrix's interface (common.hpp:48-75).
class Matrix {
 public:
  Matrix() = default;
  Matrix(int r, int c) : r_(r), c_(c), d_(static_cast<size_t>(r) * c, 0.0) {}
  int rows() const { return r_; }
  int cols() const { return c_; }
  double& operator()(int r, int c) { return d_[static_cast<size_t>(r) * c_ + c]; }
  double operator()(int r, int c) const { return d_[static_cast<size_t>(r) * c_ + c]; }
  const double* data() const { return d_.data(); }
  bool empty() const { return d_.empty(); }

 private:
  int r_ = 0, c_ = 0;
  std::vector<double> d_;
};

}  // namespace

int main() {
  orc_rng rng{1234};
  int failures = 0;
  const int A = 29;
  std::vector<Matrix> batch;
  std::vector<std::vector<int>> labels;
  for (int i = 0; i < 6; ++i) {
    const int T = 40 + 30 * i, L = 10 + 5 * i;
    Matrix x(T, A);
    for (int t = 0; t < T; ++t)
      for (int k = 0; k < A; ++k) x(t, k) = static_cast<float>(orc_rng_normal(&rng));
    std::vector<int> lab(L);
    for (int& c : lab) c = static_cast<int>(orc_rng_below(&rng, A - 1));
    batch.push_back(x);
    labels.push_back(lab);
  }
  labels[5] = std::vector<int>(200, 3);  // infeasible: T=190 < min_frames=399
  std::vector<Matrix> dl;
  auto costs = ds2ctc::ctc_loss_batch_gpu(batch, labels, A - 1, &dl);
  for (size_t i = 0; i < batch.size(); ++i) {
    const Matrix& x = batch[i];
    std::vector<double> g(static_cast<size_t>(x.rows()) * A);
    double loss = 0;
    const int ok = orc_ctc_loss(x.data(), x.rows(), A, labels[i].data(), static_cast<int>(labels[i].size()), A - 1,
                                &loss, g.data());
    auto one = ds2ctc::ctc_loss_gpu(x, labels[i], A - 1);
    if (ok != static_cast<int>(one.feasible) || ok != static_cast<int>(std::isfinite(costs[i]))) {
      std::printf("utt %zu: feasibility mismatch\n", i);
      ++failures;
      continue;
    }
    if (!ok) {
      for (int t = 0; t < x.rows(); ++t)
        for (int k = 0; k < A; ++k)
          if (dl[i](t, k) != 0.0) ++failures;
      continue;
    }
    double gerr = 0, gerr1 = 0;
    for (int t = 0; t < x.rows(); ++t)
      for (int k = 0; k < A; ++k) {
        gerr = std::fmax(gerr, std::fabs(dl[i](t, k) - g[static_cast<size_t>(t) * A + k]));
        gerr1 = std::fmax(gerr1, std::fabs(one.logit_grad(t, k) - g[static_cast<size_t>(t) * A + k]));
      }
    const double rel = std::fabs(costs[i] - loss) / loss, rel1 = std::fabs(one.loss - loss) / loss;
    std::printf("utt %zu T=%d L=%zu loss %.6f gpu %.6f rel %.2e grad %.2e | single rel %.2e grad %.2e\n", i,
                x.rows(), labels[i].size(), loss, costs[i], rel, gerr, rel1, gerr1);
    if (rel > 1e-4 || gerr > 1e-4 || rel1 > 1e-4 || gerr1 > 1e-4) ++failures;
  }
  // viterbi_align_gpu / ctc_lattice_gpu (the f2 / f3 drop-ins) vs the oracle
  for (size_t i = 0; i < 5; ++i) {
    const Matrix& x = batch[i];
    const int T = x.rows(), L = static_cast<int>(labels[i].size()), S = 2 * L + 1;
    std::vector<int> ref(static_cast<size_t>(T));
    const int rc = orc_viterbi_align(x.data(), T, A, labels[i].data(), L, A - 1, ref.data());
    try {
      const std::vector<int> al = ds2ctc::viterbi_align_gpu(x, labels[i], A - 1);
      if (rc != 0 || al != ref) {
        std::printf("utt %zu: alignment differs\n", i);
        ++failures;
      }
    } catch (const std::exception& e) {
      if (rc == 0) {
        std::printf("utt %zu: unexpected throw %s\n", i, e.what());
        ++failures;
      }
    }
    std::vector<double> ra(static_cast<size_t>(S) * T), rb(ra.size());
    double rlp = 0;
    orc_ctc_lattice(x.data(), T, A, labels[i].data(), L, A - 1, ra.data(), rb.data(), &rlp);
    const auto lat = ds2ctc::ctc_lattice_gpu(x, labels[i], A - 1);
    double err = std::fabs(lat.log_prob - rlp);
    for (int s = 0; s < S; ++s)
      for (int t = 0; t < T; ++t) {
        const double r1 = ra[static_cast<size_t>(s) * T + t], r2 = rb[static_cast<size_t>(s) * T + t];
        if (std::isinf(r1) != std::isinf(lat.alpha(s, t)) || std::isinf(r2) != std::isinf(lat.beta(s, t))) ++failures;
        if (std::isfinite(r1)) err = std::fmax(err, std::fabs(lat.alpha(s, t) - r1));
        if (std::isfinite(r2)) err = std::fmax(err, std::fabs(lat.beta(s, t) - r2));
      }
    std::printf("utt %zu: viterbi %s, lattice max err %.2e\n", i, rc == 0 ? "aligned" : "none", err);
    if (err > 1e-9) ++failures;
  }
  std::printf("%s\n", failures ? "FAIL" : "PASS");
  return failures ? 1 : 0;
}
