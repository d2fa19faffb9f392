// The literal drop-in check: the reference's OWN types (asr::Matrix,
// asr::ctc::CtcResult, asr::ctc::CtcLattice from
// /root/reference/proj/include/asr/{common,ctc}.hpp) flow through the C++
// shim (include/ds2ctc.hpp) into the sm_100a kernels, on the cases of the
// reference's own CTC test file (proj/tests/test_ctc.cpp), at fp32
// tolerances. The checkers are the reference itself -- ctc_loss_reference /
// ctc_lattice / viterbi_align linked from its sources -- and its test
// oracles (proj/tests/oracles.hpp: brute-force path sums and Viterbi
// argmax). Test infrastructure: built only where /root/reference exists
// (tests/cpp/Makefile), run on the GPU box by tests/test_gpu_cpp.py.
//
// Every call site below is written the way a reference caller is, with the
// entry point's name the only change:
//   asr::ctc::CtcResult r = ds2ctc::ctc_loss_gpu(lp, label, blank);
#include <cmath>
#include <cstdio>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "asr/common.hpp"
#include "asr/ctc.hpp"
#include "ds2ctc.hpp"
#include "oracles.hpp"

using asr::Matrix;
using asr::Rng;

namespace {

int g_checks = 0, g_fail = 0;

void check(bool ok, const std::string& what) {
  ++g_checks;
  if (!ok) {
    ++g_fail;
    std::printf("FAIL %s\n", what.c_str());
  }
}

bool close_rel(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

// test_ctc.cpp's generators (row-normalised random log-probabilities and a
// random label of length <= max_len), drawn from the reference's own Rng.
Matrix random_logprobs(Rng& rng, int frames, int symbols) {
  Matrix m(frames, symbols);
  for (int t = 0; t < frames; ++t) {
    double z = 0;
    for (int k = 0; k < symbols; ++k) z += (m(t, k) = 0.05 + rng.uniform());
    for (int k = 0; k < symbols; ++k) m(t, k) = std::log(m(t, k) / z);
  }
  return m;
}

// The GPU sees fp32 logits (the C-ABI contract); the reference checkers get
// the same values widened back to fp64.
Matrix f32(const Matrix& x) {
  Matrix y(x.rows(), x.cols());
  for (int t = 0; t < x.rows(); ++t)
    for (int k = 0; k < x.cols(); ++k) y(t, k) = static_cast<float>(x(t, k));
  return y;
}

Matrix exp_of(const Matrix& lp) {
  Matrix p(lp.rows(), lp.cols());
  for (int t = 0; t < p.rows(); ++t)
    for (int k = 0; k < p.cols(); ++k) p(t, k) = std::exp(lp(t, k));
  return p;
}

std::vector<int> random_label(Rng& rng, int max_len, int alphabet) {
  std::vector<int> label(static_cast<size_t>(rng.below(max_len + 1)));
  for (int& c : label) c = static_cast<int>(rng.below(alphabet));
  return label;
}

// GPU result vs the reference's own ctc_loss_reference on the same logits.
void vs_reference(const Matrix& x, const std::vector<int>& label, int blank, const std::string& what) {
  const asr::ctc::CtcResult ref = asr::ctc::ctc_loss_reference(x, label, blank);
  const asr::ctc::CtcResult gpu = ds2ctc::ctc_loss_gpu(x, label, blank);  // the drop-in call
  check(gpu.feasible == ref.feasible, what + ": feasibility");
  if (!ref.feasible) {
    check(std::isinf(gpu.loss) && gpu.logit_grad.empty(), what + ": infeasible convention");
    return;
  }
  check(close_rel(gpu.loss, ref.loss, 1e-5), what + ": loss " + std::to_string(gpu.loss) + " vs " +
                                                 std::to_string(ref.loss));
  check(gpu.logit_grad.same_shape(ref.logit_grad), what + ": gradient shape");
  double worst = 0;
  for (int t = 0; t < ref.logit_grad.rows(); ++t)
    for (int k = 0; k < ref.logit_grad.cols(); ++k)
      worst = std::max(worst, std::abs(gpu.logit_grad(t, k) - ref.logit_grad(t, k)));
  check(worst <= 1e-5, what + ": gradient err " + std::to_string(worst));
}

}  // namespace

int main() {
  // test_ctc.cpp:71-79 -- T = 1, one alignment: loss = ln 2
  {
    Matrix lp(1, 2);
    lp(0, 0) = lp(0, 1) = std::log(0.5);
    asr::ctc::CtcResult r = ds2ctc::ctc_loss_gpu(lp, {0}, 1);
    check(r.feasible && close_rel(r.loss, -std::log(0.5), 1e-6), "single-frame loss");
    vs_reference(lp, {0}, 1, "single-frame");
  }
  // test_ctc.cpp:81-93 -- T = 2, label "a": p = 3/4 = the brute-force path sum
  {
    Matrix lp(2, 2, std::log(0.5));
    asr::ctc::CtcResult r = ds2ctc::ctc_loss_gpu(lp, {0}, 1);
    check(r.feasible && close_rel(std::exp(-r.loss), 0.75, 1e-6), "two-frame p = 0.75");
    check(close_rel(std::exp(-r.loss), oracle::brute_force_path_sum(exp_of(lp), {0}, 1), 1e-6), "two-frame brute");
  }
  // test_ctc.cpp:95-105 -- a repeat needs a separating blank: infeasible at T = 2
  {
    Matrix lp(2, 2, std::log(0.5));
    asr::ctc::CtcResult r = ds2ctc::ctc_loss_gpu(lp, {0, 0}, 1);
    check(!r.feasible && std::isinf(r.loss) && r.logit_grad.empty(), "repeat infeasible at T=2");
    check(asr::ctc::min_frames({0, 0}) == 3, "min_frames({0,0}) == 3");
    Matrix lp3(3, 2, std::log(0.5));
    check(static_cast<asr::ctc::CtcResult>(ds2ctc::ctc_loss_gpu(lp3, {0, 0}, 1)).feasible, "repeat feasible at T=3");
  }
  // test_ctc.cpp:107-124 -- 120 fuzzed utterances vs brute-force enumeration (same seed / stream)
  {
    Rng rng(20260808);
    for (int it = 0; it < 120; ++it) {
      const int alphabet = 1 + static_cast<int>(rng.below(3));
      const int frames = 1 + static_cast<int>(rng.below(6));
      const std::vector<int> label = random_label(rng, 3, alphabet);
      const Matrix lp = f32(random_logprobs(rng, frames, alphabet + 1));
      const double brute = oracle::brute_force_path_sum(exp_of(lp), label, alphabet);
      asr::ctc::CtcResult r = ds2ctc::ctc_loss_gpu(lp, label, alphabet);
      const std::string what = "fuzz " + std::to_string(it);
      if (frames < asr::ctc::min_frames(label)) {
        check(!r.feasible, what + ": infeasible");
        continue;
      }
      check(r.feasible && close_rel(std::exp(-r.loss), brute, 1e-5), what + ": p vs brute force");
      vs_reference(lp, label, alphabet, what);
    }
  }
  // test_ctc.cpp:126-147 -- gradients through the softmax on logits in [-1, 1)
  // (the reference checks its own against finite differences; here the GPU's
  // against the reference's, same seed and generator)
  {
    Rng rng(7);
    for (int it = 0; it < 12; ++it) {
      const int alphabet = 1 + static_cast<int>(rng.below(3));
      const int frames = 2 + static_cast<int>(rng.below(4));
      std::vector<int> label = random_label(rng, 2, alphabet);
      while (!label.empty() && frames < asr::ctc::min_frames(label)) label.pop_back();
      Matrix logits(frames, alphabet + 1);
      for (int t = 0; t < frames; ++t)
        for (int k = 0; k <= alphabet; ++k) logits(t, k) = rng.uniform(-1.0, 1.0);
      vs_reference(f32(logits), label, alphabet, "grad " + std::to_string(it));
    }
  }
  // test_ctc.cpp:172-199 -- lattice export: invalid cells are -inf after the
  // alpha + beta combine, valid ones finite (enumeration oracle)
  {
    Rng rng(31337);
    for (int it = 0; it < 40; ++it) {
      const int alphabet = 1 + static_cast<int>(rng.below(3));
      const int frames = 1 + static_cast<int>(rng.below(6));
      const std::vector<int> label = random_label(rng, 3, alphabet);
      if (frames < asr::ctc::min_frames(label)) continue;
      const Matrix lp = f32(random_logprobs(rng, frames, alphabet + 1));
      asr::ctc::CtcLattice lat = ds2ctc::ctc_lattice_gpu(lp, label, alphabet);  // the drop-in call
      const asr::ctc::CtcLattice ref = asr::ctc::ctc_lattice(lp, label, alphabet);
      check(lat.augmented_label == ref.augmented_label, "lattice aug " + std::to_string(it));
      std::set<std::pair<int, int>> valid;
      for (const auto& rows : oracle::enumerate_row_paths(frames, lat.augmented_label, alphabet))
        for (int t = 0; t < frames; ++t) valid.insert({rows[t], t});
      for (int s = 0; s < lat.alpha.rows(); ++s)
        for (int t = 0; t < frames; ++t) {
          const double comb = lat.alpha(s, t) + lat.beta(s, t);
          check(valid.count({s, t}) ? std::isfinite(comb) : comb == asr::kNegInf,
                "lattice cancellation " + std::to_string(it));
        }
      check(close_rel(lat.log_prob, ref.log_prob, 1e-12), "lattice log p " + std::to_string(it));
    }
  }
  // test_ctc.cpp:277-284 -- lattice TSV dump: the reference's printer and the
  // shim's (on the GPU lattice) write the same text for the test's lattice
  // (values within 1e-12, printed at the stream's default precision)
  {
    Matrix lp(3, 3, std::log(1.0 / 3));
    const auto lat = ds2ctc::ctc_lattice_gpu(lp, {0}, 2);
    std::ostringstream mine, theirs;
    ds2ctc::dump_lattice_tsv(lat, mine);
    asr::ctc::dump_lattice_tsv(asr::ctc::ctc_lattice(lp, {0}, 2), theirs);
    check(mine.str().find("# alpha (3 x 3)") != std::string::npos, "tsv alpha header");
    check(mine.str().find("# beta (3 x 3)") != std::string::npos, "tsv beta header");
    check(mine.str() == theirs.str(), "tsv text equals the reference's");
    std::ostringstream conv;  // through the conversion to the reference's lattice type
    asr::ctc::dump_lattice_tsv(static_cast<asr::ctc::CtcLattice>(lat), conv);
    check(conv.str() == theirs.str(), "tsv via asr::ctc::CtcLattice");
  }
  // test_ctc.cpp:233-241 -- Viterbi: forced one-to-one alignment
  {
    Matrix lp(3, 4, std::log(0.02));
    const std::vector<int> label = {2, 0, 1};
    for (int t = 0; t < 3; ++t) lp(t, label[t]) = std::log(0.94);
    check(ds2ctc::viterbi_align_gpu(lp, label, 3) == label, "viterbi forced");
  }
  // test_ctc.cpp:243-256 -- Viterbi vs brute-force argmax with the tie rule
  {
    Rng rng(4242);
    for (int it = 0; it < 80; ++it) {
      const int alphabet = 1 + static_cast<int>(rng.below(3));
      const int frames = 1 + static_cast<int>(rng.below(6));
      const std::vector<int> label = random_label(rng, 3, alphabet);
      if (frames < asr::ctc::min_frames(label)) continue;
      const Matrix lp = f32(random_logprobs(rng, frames, alphabet + 1));
      const std::vector<int> got = ds2ctc::viterbi_align_gpu(lp, label, alphabet);
      check(got == oracle::brute_force_viterbi(exp_of(lp), label, alphabet), "viterbi brute " + std::to_string(it));
      check(got == asr::ctc::viterbi_align(lp, label, alphabet), "viterbi ref " + std::to_string(it));
      check(oracle::collapse(got, alphabet) == label, "viterbi collapse " + std::to_string(it));
    }
  }
  // test_ctc.cpp:258-266 -- Viterbi tie prefers staying over advancing
  {
    Matrix lp(2, 2, std::log(0.5));
    check(ds2ctc::viterbi_align_gpu(lp, {0}, 1) == std::vector<int>({0, 1}), "viterbi tie");
  }
  // test_ctc.cpp:268-275 -- empty label: loss = 4 ln 3, all-blank alignment
  {
    Matrix lp(4, 3, std::log(1.0 / 3));
    asr::ctc::CtcResult r = ds2ctc::ctc_loss_gpu(lp, {}, 2);
    check(r.feasible && close_rel(r.loss, 4 * std::log(3.0), 1e-6), "empty label loss");
    check(ds2ctc::viterbi_align_gpu(lp, {}, 2) == std::vector<int>(4, 2), "empty label alignment");
  }
  // The trainer's batched loop (trainer.cpp:155-171) through the batched shim
  // with asr::Matrix batches: every utterance vs ctc_loss_reference.
  {
    Rng rng(1234);
    std::vector<Matrix> batch;
    std::vector<std::vector<int>> labels;
    for (int i = 0; i < 8; ++i) {
      const int T = 30 + 17 * i, L = 5 + 3 * i;
      Matrix x(T, 29);
      for (int t = 0; t < T; ++t)
        for (int k = 0; k < 29; ++k) x(t, k) = static_cast<float>(rng.normal());
      std::vector<int> lab(static_cast<size_t>(L));
      for (int& c : lab) c = static_cast<int>(rng.below(28));
      batch.push_back(x);
      labels.push_back(lab);
    }
    labels[7] = std::vector<int>(120, 4);  // T = 149 < min_frames = 239: skipped, zero gradient
    std::vector<Matrix> dlogits;
    const std::vector<double> costs = ds2ctc::ctc_loss_batch_gpu(batch, labels, 28, &dlogits);
    for (size_t i = 0; i < batch.size(); ++i) {
      const asr::ctc::CtcResult ref = asr::ctc::ctc_loss_reference(batch[i], labels[i], 28);
      const std::string what = "batch " + std::to_string(i);
      if (!ref.feasible) {
        bool zero = true;
        for (int t = 0; t < dlogits[i].rows(); ++t)
          for (int k = 0; k < 29; ++k) zero = zero && dlogits[i](t, k) == 0.0;
        check(std::isinf(costs[i]) && zero, what + ": skipped with zero gradient");
        continue;
      }
      check(close_rel(costs[i], ref.loss, 1e-5), what + ": loss");
      double worst = 0;
      for (int t = 0; t < ref.logit_grad.rows(); ++t)
        for (int k = 0; k < 29; ++k) worst = std::max(worst, std::abs(dlogits[i](t, k) - ref.logit_grad(t, k)));
      check(worst <= 1e-5, what + ": gradient err " + std::to_string(worst));
    }
  }
  std::printf("%s: %d checks, %d failures\n", g_fail ? "FAILED" : "PASS", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
