/*
 * ctc_oracle.c -- fp64 CPU restatement of the reference CTC path.
 *
 * TEST INFRASTRUCTURE ONLY (see ctc_oracle.h). Every function follows the
 * cited reference file:line operation-for-operation (same order of floating
 * point operations, same libm calls), so on x86-64 it reproduces the
 * reference's default fp64 build bit for bit; tests/test_oracle.py pins that.
 */
#include "ctc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define NEG_INF (-INFINITY)

/* ref: proj/include/asr/ctc.hpp:30-35 */
double orc_log_sum_exp_guarded(double a, double b) {
  if (a == NEG_INF) return b;
  if (b == NEG_INF) return a;
  if (a < b) {
    double t = a;
    a = b;
    b = t;
  }
  return a + log1p(exp(b - a));
}

/* ref: proj/src/ctc.cpp:24-37 (std::max(mx, v) keeps mx unless mx < v) */
void orc_log_softmax_rows(const double* logits, int rows, int cols, double* out) {
  for (int t = 0; t < rows; ++t) {
    const double* in = logits + (size_t)t * cols;
    double* o = out + (size_t)t * cols;
    double mx = in[0];
    for (int k = 1; k < cols; ++k)
      if (mx < in[k]) mx = in[k];
    double sum = 0;
    for (int k = 0; k < cols; ++k) sum += exp(in[k] - mx);
    double lse = mx + log(sum);
    for (int k = 0; k < cols; ++k) o[k] = in[k] - lse;
  }
}

/* ref: proj/src/ctc.cpp:41-43 */
static int skip_allowed(const int* aug, int blank, int s) {
  return s >= 2 && aug[s] != blank && aug[s] != aug[s - 2];
}

/* ref: proj/src/ctc.cpp:91-100 */
void orc_augment_label(const int* label, int L, int blank, int* aug) {
  aug[0] = blank;
  for (int i = 0; i < L; ++i) {
    aug[2 * i + 1] = label[i];
    aug[2 * i + 2] = blank;
  }
}

/* ref: proj/src/ctc.cpp:102-107 */
int orc_min_frames(const int* label, int L) {
  int needed = L;
  for (int i = 1; i < L; ++i)
    if (label[i] == label[i - 1]) ++needed;
  return needed;
}

/* ref: proj/src/ctc.cpp:109-124 */
void orc_forward_column(const double* logprobs, int cols, const int* aug, int S, int blank, int t,
                        const double* prev, double* out) {
  const double* lp = logprobs + (size_t)t * cols;
  if (t == 0) {
    for (int s = 0; s < S; ++s) out[s] = s < 2 ? lp[aug[s]] : NEG_INF;
    return;
  }
  for (int s = 0; s < S; ++s) {
    double acc = prev[s];
    if (s >= 1) acc = orc_log_sum_exp_guarded(acc, prev[s - 1]);
    if (skip_allowed(aug, blank, s)) acc = orc_log_sum_exp_guarded(acc, prev[s - 2]);
    out[s] = acc == NEG_INF ? NEG_INF : acc + lp[aug[s]];
  }
}

/* ref: proj/src/ctc.cpp:126-143 */
void orc_backward_column(const double* logprobs, int rows, int cols, const int* aug, int S, int blank,
                         int t, const double* next, double* out) {
  if (t == rows - 1) {
    for (int s = 0; s < S; ++s) out[s] = s >= S - 2 ? 0 : NEG_INF;
    return;
  }
  const double* lp = logprobs + (size_t)(t + 1) * cols;
  for (int s = 0; s < S; ++s) {
    double acc = next[s] == NEG_INF ? NEG_INF : next[s] + lp[aug[s]];
    if (s + 1 < S && next[s + 1] != NEG_INF)
      acc = orc_log_sum_exp_guarded(acc, next[s + 1] + lp[aug[s + 1]]);
    if (s + 2 < S && skip_allowed(aug, blank, s + 2) && next[s + 2] != NEG_INF)
      acc = orc_log_sum_exp_guarded(acc, next[s + 2] + lp[aug[s + 2]]);
    out[s] = acc;
  }
}

/* ref: proj/src/ctc.cpp:81-87 */
static double final_log_prob(const double* last_alpha, int S) {
  double lp = NEG_INF;
  if (S >= 2) lp = orc_log_sum_exp_guarded(lp, last_alpha[S - 2]);
  lp = orc_log_sum_exp_guarded(lp, last_alpha[S - 1]);
  return lp;
}

/* KeyGroups as a CSR over (symbol, row) pairs sorted ascending. ref: proj/src/ctc.cpp:47-66 */
typedef struct {
  int nkeys;
  int* keys;   /* distinct symbols ascending */
  int* start;  /* nkeys + 1 */
  int* rows;   /* S rows, ascending within a key */
} key_groups;

static int cmp_pair(const void* pa, const void* pb) {
  const int* a = (const int*)pa;
  const int* b = (const int*)pb;
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
  return 0;
}

static void group_rows_by_key(const int* aug, int S, key_groups* g) {
  int* kv = (int*)malloc(sizeof(int) * 2 * (size_t)S);
  for (int s = 0; s < S; ++s) {
    kv[2 * s] = aug[s];
    kv[2 * s + 1] = s;
  }
  qsort(kv, (size_t)S, 2 * sizeof(int), cmp_pair);
  g->keys = (int*)malloc(sizeof(int) * (size_t)S);
  g->start = (int*)malloc(sizeof(int) * ((size_t)S + 1));
  g->rows = (int*)malloc(sizeof(int) * (size_t)S);
  g->nkeys = 0;
  for (int i = 0; i < S; ++i) {
    if (g->nkeys == 0 || g->keys[g->nkeys - 1] != kv[2 * i]) {
      g->keys[g->nkeys] = kv[2 * i];
      g->start[g->nkeys] = i;
      g->nkeys++;
    }
    g->rows[i] = kv[2 * i + 1];
  }
  g->start[g->nkeys] = S;
  free(kv);
}

static void free_groups(key_groups* g) {
  free(g->keys);
  free(g->start);
  free(g->rows);
}

/* ref: proj/src/ctc.cpp:69-79 */
static void grad_column(const double* logprobs, int cols, const key_groups* g, double log_prob,
                        const double* gamma, int t, double* grad) {
  const double* lp = logprobs + (size_t)t * cols;
  double* gr = grad + (size_t)t * cols;
  for (int k = 0; k < cols; ++k) gr[k] = exp(lp[k]);
  for (int i = 0; i < g->nkeys; ++i) {
    double acc = NEG_INF;
    for (int j = g->start[i]; j < g->start[i + 1]; ++j) acc = orc_log_sum_exp_guarded(acc, gamma[g->rows[j]]);
    gr[g->keys[i]] -= exp(acc - log_prob);
  }
}

/* ref: proj/src/ctc.cpp:171-207 */
int orc_ctc_loss(const double* logits, int T, int C, const int* label, int L, int blank, double* loss,
                 double* grad) {
  *loss = INFINITY;
  if (T < orc_min_frames(label, L)) return 0; /* ctc.cpp:173 */
  if (T == 0) {                              /* L == 0 here; reference UB (ctc.cpp:81-86) */
    *loss = 0.0;
    return 1;
  }
  int S = 2 * L + 1;
  double* logprobs = (double*)malloc(sizeof(double) * (size_t)T * C);
  int* aug = (int*)malloc(sizeof(int) * (size_t)S);
  double* alpha = (double*)malloc(sizeof(double) * (size_t)S * T); /* alpha(s, t) at s*T + t */
  double* prev = (double*)malloc(sizeof(double) * (size_t)S);
  double* cur = (double*)malloc(sizeof(double) * (size_t)S);
  orc_log_softmax_rows(logits, T, C, logprobs);
  orc_augment_label(label, L, blank, aug);
  for (int t = 0; t < T; ++t) {
    orc_forward_column(logprobs, C, aug, S, blank, t, prev, cur);
    for (int s = 0; s < S; ++s) alpha[(size_t)s * T + t] = cur[s];
    double* tmp = prev;
    prev = cur;
    cur = tmp;
  }
  double log_prob = final_log_prob(prev, S);
  int feasible = 0;
  if (log_prob != NEG_INF) { /* ctc.cpp:189-193 */
    feasible = 1;
    if (grad) {
      key_groups g;
      group_rows_by_key(aug, S, &g);
      double* beta_next = prev; /* ignored at t == T-1 */
      double* beta_t = cur;
      double* gamma = (double*)malloc(sizeof(double) * (size_t)S);
      for (int t = T - 1; t >= 0; --t) {
        orc_backward_column(logprobs, T, C, aug, S, blank, t, beta_next, beta_t);
        for (int s = 0; s < S; ++s) gamma[s] = alpha[(size_t)s * T + t] + beta_t[s];
        grad_column(logprobs, C, &g, log_prob, gamma, t, grad);
        double* tmp = beta_next;
        beta_next = beta_t;
        beta_t = tmp;
      }
      prev = beta_next;
      cur = beta_t;
      free(gamma);
      free_groups(&g);
    }
    *loss = -log_prob;
  }
  free(logprobs);
  free(aug);
  free(alpha);
  free(prev);
  free(cur);
  return feasible;
}

/* ref: proj/src/ctc.cpp:145-169 */
void orc_ctc_lattice(const double* logits, int T, int C, const int* label, int L, int blank,
                     double* alpha, double* beta, double* log_prob) {
  int S = 2 * L + 1;
  double* logprobs = (double*)malloc(sizeof(double) * (size_t)T * C);
  int* aug = (int*)malloc(sizeof(int) * (size_t)S);
  double* prev = (double*)malloc(sizeof(double) * (size_t)S);
  double* cur = (double*)malloc(sizeof(double) * (size_t)S);
  orc_log_softmax_rows(logits, T, C, logprobs);
  orc_augment_label(label, L, blank, aug);
  for (int t = 0; t < T; ++t) {
    orc_forward_column(logprobs, C, aug, S, blank, t, prev, cur);
    for (int s = 0; s < S; ++s) alpha[(size_t)s * T + t] = cur[s];
    double* tmp = prev;
    prev = cur;
    cur = tmp;
  }
  *log_prob = final_log_prob(prev, S);
  for (int t = T - 1; t >= 0; --t) {
    orc_backward_column(logprobs, T, C, aug, S, blank, t, prev, cur);
    for (int s = 0; s < S; ++s) beta[(size_t)s * T + t] = cur[s];
    double* tmp = prev;
    prev = cur;
    cur = tmp;
  }
  free(logprobs);
  free(aug);
  free(prev);
  free(cur);
}

/* ref: proj/src/ctc.cpp:327-370 */
int orc_viterbi_align(const double* logits, int T, int C, const int* label, int L, int blank, int* out) {
  if (T < orc_min_frames(label, L) || T == 0) return -1;
  int S = 2 * L + 1;
  double* logprobs = (double*)malloc(sizeof(double) * (size_t)T * C);
  int* aug = (int*)malloc(sizeof(int) * (size_t)S);
  double* score = (double*)malloc(sizeof(double) * (size_t)S * T);
  int* from = (int*)malloc(sizeof(int) * (size_t)S * T);
  orc_log_softmax_rows(logits, T, C, logprobs);
  orc_augment_label(label, L, blank, aug);
  for (size_t i = 0; i < (size_t)S * T; ++i) {
    score[i] = NEG_INF;
    from[i] = -1;
  }
#define SC(s, t) score[(size_t)(s) * T + (t)]
  for (int s = 0; s < (S < 2 ? S : 2); ++s) SC(s, 0) = logprobs[aug[s]];
  for (int t = 1; t < T; ++t) {
    const double* lp = logprobs + (size_t)t * C;
    for (int s = 0; s < S; ++s) {
      double best = SC(s, t - 1);
      int pred = s;
      if (s >= 1 && SC(s - 1, t - 1) > best) {
        best = SC(s - 1, t - 1);
        pred = s - 1;
      }
      if (skip_allowed(aug, blank, s) && SC(s - 2, t - 1) > best) {
        best = SC(s - 2, t - 1);
        pred = s - 2;
      }
      if (best == NEG_INF) continue;
      SC(s, t) = best + lp[aug[s]];
      from[(size_t)s * T + t] = pred;
    }
  }
  int end = S - 1;
  if (S >= 2 && SC(S - 2, T - 1) > SC(end, T - 1)) end = S - 2;
  int rc = 0;
  if (SC(end, T - 1) == NEG_INF) {
    rc = -1;
  } else {
    int s = end;
    for (int t = T - 1; t >= 0; --t) {
      out[t] = aug[s];
      s = from[(size_t)s * T + t];
    }
  }
#undef SC
  free(logprobs);
  free(aug);
  free(score);
  free(from);
  return rc;
}

/* ---- batched wrapper (trainer convention, proj/src/trainer.cpp:158-169) ---- */

typedef struct {
  const float* acts;
  const int* flat_labels;
  const int* label_offsets;
  const int* label_lengths;
  const int* input_lengths;
  int A, B, blank, Tmax;
  double* costs;
  double* grads;
  int next; /* guarded by mu */
  pthread_mutex_t mu;
} batch_job;

static void run_one(batch_job* job, int b) {
  int T = job->input_lengths[b];
  int A = job->A;
  int L = job->label_lengths[b];
  const int* label = job->flat_labels + job->label_offsets[b];
  double* x = (double*)malloc(sizeof(double) * ((size_t)T * A + 1));
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < A; ++k) x[(size_t)t * A + k] = (double)job->acts[((size_t)t * job->B + b) * A + k];
  double* g = job->grads ? (double*)calloc((size_t)T * A + 1, sizeof(double)) : NULL;
  double loss;
  int ok = orc_ctc_loss(x, T, A, label, L, job->blank, &loss, g);
  job->costs[b] = ok ? loss : INFINITY;
  if (job->grads) {
    for (int t = 0; t < job->Tmax; ++t)
      for (int k = 0; k < A; ++k)
        job->grads[((size_t)t * job->B + b) * A + k] = (ok && t < T) ? g[(size_t)t * A + k] : 0.0;
    free(g);
  }
  free(x);
}

static void* batch_worker(void* arg) {
  batch_job* job = (batch_job*)arg;
  for (;;) {
    pthread_mutex_lock(&job->mu);
    int b = job->next++;
    pthread_mutex_unlock(&job->mu);
    if (b >= job->B) break;
    run_one(job, b);
  }
  return NULL;
}

void orc_ctc_batch(const float* activations, const int* flat_labels, const int* label_lengths,
                   const int* input_lengths, int alphabet_size, int minibatch, int blank,
                   double* costs, double* grads, int nthreads) {
  batch_job job;
  int* offs = (int*)malloc(sizeof(int) * ((size_t)minibatch + 1));
  int Tmax = 0;
  offs[0] = 0;
  for (int b = 0; b < minibatch; ++b) {
    offs[b + 1] = offs[b] + label_lengths[b];
    if (input_lengths[b] > Tmax) Tmax = input_lengths[b];
  }
  job.acts = activations;
  job.flat_labels = flat_labels;
  job.label_offsets = offs;
  job.label_lengths = label_lengths;
  job.input_lengths = input_lengths;
  job.A = alphabet_size;
  job.B = minibatch;
  job.blank = blank;
  job.Tmax = Tmax;
  job.costs = costs;
  job.grads = grads;
  job.next = 0;
  pthread_mutex_init(&job.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    batch_worker(&job);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, batch_worker, &job);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
  }
  pthread_mutex_destroy(&job.mu);
  free(offs);
}

/* ---- SplitMix64, ref: proj/include/asr/common.hpp:92-118 ---- */

uint64_t orc_rng_next_u64(orc_rng* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

uint64_t orc_rng_below(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }

double orc_rng_normal(orc_rng* r) {
  double u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* ---- SortaGrad, ref: proj/src/trainer.cpp:58-91 ---- */

static const int* g_sort_lengths; /* qsort has no context argument; guarded by single-threaded use */

static int cmp_len_stable(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  int la = g_sort_lengths[a], lb = g_sort_lengths[b];
  if (la != lb) return la < lb ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0); /* stable: original index order on ties */
}

static void shuffle_i64(orc_rng* rng, int64_t* v, size_t n) {
  for (size_t i = n; i > 1; --i) {
    size_t j = (size_t)orc_rng_below(rng, i);
    int64_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

void orc_sortagrad_order(const int* lengths, int n, int global_batch, int epoch, uint64_t seed,
                         int sortagrad_on, int64_t* out) {
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  for (int i = 0; i < n; ++i) idx[i] = i;
  orc_rng rng = {seed * 0x9e3779b9ULL + (uint64_t)epoch + 1};
  if (!sortagrad_on) {
    shuffle_i64(&rng, idx, (size_t)n);
    memcpy(out, idx, sizeof(int64_t) * (size_t)n);
    free(idx);
    return;
  }
  g_sort_lengths = lengths;
  qsort(idx, (size_t)n, sizeof(int64_t), cmp_len_stable);
  if (epoch == 0) {
    memcpy(out, idx, sizeof(int64_t) * (size_t)n);
    free(idx);
    return;
  }
  size_t batches = ((size_t)n + global_batch - 1) / global_batch;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (batches + 1));
  for (size_t i = 0; i < batches; ++i) order[i] = (int64_t)i;
  shuffle_i64(&rng, order, batches);
  size_t k = 0;
  for (size_t bi = 0; bi < batches; ++bi) {
    size_t begin = (size_t)order[bi] * global_batch;
    size_t end = begin + global_batch < (size_t)n ? begin + global_batch : (size_t)n;
    for (size_t i = begin; i < end; ++i) out[k++] = idx[i];
  }
  free(order);
  free(idx);
}
