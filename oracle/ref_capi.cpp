// ref_capi.cpp -- extern "C" shim over the reference's OWN fp64 CTC build.
//
// TEST / BASELINE INFRASTRUCTURE. oracle/Makefile compiles this file together
// with the unmodified reference sources where they lie
// (/root/reference/proj/src/{ctc,common,trainer,...}.cpp) into
// oracle/_ref/libasr_ref.so. Nothing here re-implements CTC: every entry point
// forwards to the reference's functions so tests can (a) pin the oracle
// restatement (oracle/ctc_oracle.c) and the golden fixtures to the real
// reference, and (b) time the reference CPU CTC as bench.py's cpu_baseline and
// --impl reference arm (threaded the way the paper's CPU CTC was: one
// utterance per thread; serially per utterance as
// trainer.cpp:158-169 calls it when nthreads == 1).
#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "asr/common.hpp"
#include "asr/ctc.hpp"
#include "asr/nn.hpp"
#include "asr/trainer.hpp"

using asr::Matrix;

namespace {

Matrix widen(const double* x, int rows, int cols) {
  Matrix m(rows, cols);
  for (int i = 0; i < rows * cols; ++i) m.data()[i] = x[i];
  return m;
}

}  // namespace

extern "C" {

// asr::ctc::ctc_loss_reference (ctc.cpp:171-207). Returns feasible; grad (T x C) written if feasible.
int ref_ctc_loss(const double* logits, int T, int C, const int* label, int L, int blank, double* loss,
                 double* grad) {
  Matrix x = widen(logits, T, C);
  std::vector<int> lab(label, label + L);
  auto res = asr::ctc::ctc_loss_reference(x, lab, blank);
  *loss = res.loss;
  if (res.feasible && grad)
    for (int i = 0; i < T * C; ++i) grad[i] = res.logit_grad.data()[i];
  return res.feasible ? 1 : 0;
}

// asr::ctc::ctc_loss_parallel (ctc.cpp:209-325).
int ref_ctc_loss_parallel(const double* logits, int T, int C, const int* label, int L, int blank, int workers,
                          double* loss, double* grad) {
  Matrix x = widen(logits, T, C);
  std::vector<int> lab(label, label + L);
  auto res = asr::ctc::ctc_loss_parallel(x, lab, blank, workers);
  *loss = res.loss;
  if (res.feasible && grad)
    for (int i = 0; i < T * C; ++i) grad[i] = res.logit_grad.data()[i];
  return res.feasible ? 1 : 0;
}

// asr::ctc::ctc_lattice (ctc.cpp:145-169): alpha/beta S x T row-major.
void ref_ctc_lattice(const double* logits, int T, int C, const int* label, int L, int blank, double* alpha,
                     double* beta, double* log_prob) {
  Matrix x = widen(logits, T, C);
  std::vector<int> lab(label, label + L);
  auto lat = asr::ctc::ctc_lattice(x, lab, blank);
  int S = lat.alpha.rows();
  for (int i = 0; i < S * T; ++i) {
    alpha[i] = lat.alpha.data()[i];
    beta[i] = lat.beta.data()[i];
  }
  *log_prob = lat.log_prob;
}

// asr::ctc::viterbi_align (ctc.cpp:327-370). Returns 0, or -1 when the reference throws.
int ref_viterbi_align(const double* logits, int T, int C, const int* label, int L, int blank, int* out) {
  try {
    Matrix x = widen(logits, T, C);
    std::vector<int> lab(label, label + L);
    auto a = asr::ctc::viterbi_align(x, lab, blank);
    for (int t = 0; t < T; ++t) out[t] = a[t];
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_min_frames(const int* label, int L) { return asr::ctc::min_frames(std::vector<int>(label, label + L)); }

// asr::trainer::sortagrad_order (trainer.cpp:58-91).
void ref_sortagrad_order(const int* lengths, int n, int global_batch, int epoch, uint64_t seed, int sortagrad_on,
                         int64_t* out) {
  std::vector<int> len(lengths, lengths + n);
  auto order = asr::trainer::sortagrad_order(len, global_batch, epoch, seed, sortagrad_on != 0);
  for (int i = 0; i < n; ++i) out[i] = static_cast<int64_t>(order[i]);
}

// Batched driver over [Tmax][B][A] fp32 activations with the trainer's
// infeasible convention (trainer.cpp:158-169). Each utterance is widened to
// an fp64 Matrix slice and passed to ctc_loss_reference unchanged.
// nthreads threads pull utterances from a shared counter. grads may be NULL
// (cost only, as evaluate_mean_loss uses it, trainer.cpp:201-214); when
// non-NULL it receives fp32 gradients, zero on infeasible and padded rows.
void ref_ctc_batch(const float* acts, const int* flat_labels, const int* label_lengths, const int* input_lengths,
                   int A, int B, int blank, double* costs, float* grads, int nthreads) {
  std::vector<int> offs(B + 1, 0);
  int Tmax = 0;
  for (int b = 0; b < B; ++b) {
    offs[b + 1] = offs[b] + label_lengths[b];
    Tmax = std::max(Tmax, input_lengths[b]);
  }
  std::atomic<int> next{0};
  auto body = [&]() {
    for (;;) {
      int b = next.fetch_add(1);
      if (b >= B) break;
      int T = input_lengths[b];
      Matrix x(T, A);
      for (int t = 0; t < T; ++t)
        for (int k = 0; k < A; ++k) x(t, k) = acts[(static_cast<size_t>(t) * B + b) * A + k];
      std::vector<int> lab(flat_labels + offs[b], flat_labels + offs[b] + label_lengths[b]);
      asr::ctc::CtcResult res;
      if (T == 0 && lab.empty()) {
        res.feasible = true;  // reference UB (ctc.cpp:81-86); defined as loss 0 here
        res.loss = 0;
      } else {
        res = asr::ctc::ctc_loss_reference(x, lab, blank);
      }
      costs[b] = res.feasible ? res.loss : INFINITY;
      if (grads) {
        for (int t = 0; t < Tmax; ++t)
          for (int k = 0; k < A; ++k)
            grads[(static_cast<size_t>(t) * B + b) * A + k] =
                (res.feasible && t < T) ? static_cast<float>(res.logit_grad(t, k)) : 0.0f;
      }
    }
  };
  if (nthreads <= 1) {
    body();
  } else {
    std::vector<std::thread> th;
    for (int i = 0; i < nthreads; ++i) th.emplace_back(body);
    for (auto& t : th) t.join();
  }
}

// The reference's own output-layer backward: asr::nn::make_fully_connected(H, A,
// relu = false, batchnorm = false) (network.cpp:135), train-mode forward on the
// utterance matrices x[b] (T_b x H) to cache them, then backward(dlogits[b])
// (nn.cpp:874-899). Inputs are the batched [T_max][B][.] buffers; w is A x H.
// Outputs: dw (A x H), db (A), dx [T_max][B][H] (zero past T_b). fp64 throughout.
void ref_fc_backward(const float* x, const float* dlogits, const int* input_lengths, int B, int Tmax, int H, int A,
                     const float* w, double* dw, double* db, double* dx) {
  auto layer = asr::nn::make_fully_connected(H, A, false, false);
  std::vector<asr::nn::ParamRef> params;
  layer->collect("fc", params);
  for (auto& p : params) {
    if (p.value->rows() == A && p.value->cols() == H)
      for (int i = 0; i < A * H; ++i) p.value->data()[i] = w[i];
  }
  asr::nn::Batch in(B), dout(B);
  for (int b = 0; b < B; ++b) {
    const int T = input_lengths[b];
    in[b] = Matrix(T, H);
    dout[b] = Matrix(T, A);
    for (int t = 0; t < T; ++t) {
      for (int h = 0; h < H; ++h) in[b](t, h) = x[(static_cast<size_t>(t) * B + b) * H + h];
      for (int a = 0; a < A; ++a) dout[b](t, a) = dlogits[(static_cast<size_t>(t) * B + b) * A + a];
    }
  }
  layer->forward(in, /*train=*/true);
  asr::nn::Batch dxb = layer->backward(dout);
  for (auto& p : params) {
    if (p.grad->rows() == A && p.grad->cols() == H)
      for (int i = 0; i < A * H; ++i) dw[i] = p.grad->data()[i];
    else if (p.grad->rows() == 1 && p.grad->cols() == A)
      for (int i = 0; i < A; ++i) db[i] = p.grad->data()[i];
  }
  for (int t = 0; t < Tmax; ++t)
    for (int b = 0; b < B; ++b)
      for (int h = 0; h < H; ++h)
        dx[(static_cast<size_t>(t) * B + b) * H + h] = t < input_lengths[b] ? dxb[b](t, h) : 0.0;
}

}  // extern "C"
