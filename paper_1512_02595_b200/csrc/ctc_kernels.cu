// ctc_kernels.cu -- sm_100a kernels of the DS2 CTC loss + gradient.
//
// Reference semantics: asr::ctc::ctc_loss_reference (proj/src/ctc.cpp:171-207)
// per utterance, with the column-parallel lattice scheme of ctc_loss_parallel
// (ctc.cpp:209-325; paper §5.2 / PAPER.md:749-778): every cell of a column is
// computed, invalid cells hold -inf or finite garbage that cancels in the
// plain alpha+beta add (ctc.cpp:200).
//
// B200 design:
//  * The recursions run on the RAW logits. Per-frame normalisation shifts
//    every path through frame t by the same lse_t, so occupancies
//    alpha+beta-logZ are unchanged and log p = logZ - sum_t lse_t. The
//    log-softmax therefore only appears in the gradient epilogue
//    (softmax term) and the cost, never on the serial chain.
//  * log2 domain; the carried lattice value is fp64, the log-sum-exp
//    correction is fp32 MUFU (ex2/lg2.approx). fp32 carries accumulate
//    ulp(|alpha|) per step and miss 1e-4 at T >= 700.
//  * One 2-CTA cluster per utterance: CTA 0 runs alpha forward, CTA 1 runs
//    beta backward; each stores its first half of the lattice, they meet at
//    frame tm = (T-1)/2 (cluster barrier, log Z from alpha(tm)+beta(tm)),
//    and each then streams its second half, fusing gamma = alpha+beta,
//    the key-grouped occupancy and the gradient row write. The serial chain
//    is T steps instead of 2T.
#include <cuda_runtime.h>

#include <cstdint>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

constexpr double kLog2e = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;

__device__ __forceinline__ double dneg_inf() { return __longlong_as_double(0xfff0000000000000ULL); }

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// log2(2^a + 2^b + 2^c) with the reference's -inf discard rule
// (ctc.hpp:30-35 applied twice, ctc.cpp:228-230): -inf inputs contribute 0
// and an all -inf triple stays -inf.
__device__ __forceinline__ double lse3(double a, double b, double c) {
  double m = a > b ? a : b;
  m = m > c ? m : c;
  const float s = ex2_approx(static_cast<float>(a - m)) + ex2_approx(static_cast<float>(b - m)) +
                  ex2_approx(static_cast<float>(c - m));
  const double r = m + static_cast<double>(lg2_approx(s));
  return m == dneg_inf() ? m : r;
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// K1: per-frame logit statistics (max, log sum exp(x - max)), one warp per
// (t, b) row. The reference's log_softmax_rows (ctc.cpp:24-37) materialises
// T x A log-probs; here only 8 bytes per row are kept.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_rowstats(const float* __restrict__ x, float2* __restrict__ stats,
                                                  const UttDesc* __restrict__ desc, int t_max, int B, int A) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= t_max * B) return;
  const int t = row / B;
  const int b = row - t * B;
  if (t >= desc[b].T) return;
  const float* xr = x + static_cast<size_t>(row) * A;
  float m = -INFINITY;
  for (int c = lane; c < A; c += 32) m = fmaxf(m, __ldg(xr + c));
  m = warp_max_f(m);
  float s = 0.f;
  for (int c = lane; c < A; c += 32) s += expf(__ldg(xr + c) - m);
  s = warp_sum_f(s);
  if (lane == 0) stats[row] = make_float2(m, logf(s));
}

// ---------------------------------------------------------------------------
// K2/K3: alpha || beta pair with the fused gradient.
// ---------------------------------------------------------------------------
struct ChainSmem {
  double* col[2];  // lattice column double buffer, index s + 2, -inf sentinels at both ends
  int* aug;        // blank-extended label (ctc.cpp:91-100)
  int* skip;       // skip_allowed (ctc.cpp:41-43)
  float* erow;     // per-cell occupancy of the current gradient row
  float* occ;      // per-slot occupancy (slot 0 = odd rows labelled blank only)
  short* slot_of;  // symbol -> slot (fused path), -1 when absent
  double* redd;    // [32] block reduction scratch
  float* redf;     // [2][32] double-buffered warp partials of the blank occupancy
};

__device__ __forceinline__ void zero_rows(const ChainArgs& a, int b, int lo, int hi) {
  const size_t rs = static_cast<size_t>(a.B) * a.A;
  for (int t = lo; t < hi; ++t) {
    float* g = a.grad + static_cast<size_t>(t) * rs + static_cast<size_t>(b) * a.A;
    for (int c = threadIdx.x; c < a.A; c += blockDim.x) g[c] = 0.f;
  }
}

template <int K>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024) k_pair_chain(ChainArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dir = static_cast<int>(cluster_rank());  // 0: alpha forward, 1: beta backward
  const int b = a.order[blockIdx.x >> 1];
  const UttDesc u = a.desc[b];
  const int NT = blockDim.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int NW = NT >> 5;
  const bool want_grad = a.grad != nullptr;
  const bool fused = want_grad && a.occ == nullptr;
  const double NEG = dneg_inf();

  if (u.status != 0) {
    if (dir == 0 && tid == 0) {
      a.costs[b] = u.status == 2 ? 0.f : INFINITY;
      a.logz[b] = u.status == 2 ? 0.0 : NEG;
    }
    if (fused) zero_rows(a, b, dir == 0 ? 0 : a.t_max / 2, dir == 0 ? a.t_max / 2 : a.t_max);
    return;
  }

  const int T = u.T, S = u.S, tm = u.tm;
  const int cap = NT * K;
  ChainSmem sm;
  {
    unsigned char* p = smem_raw;
    sm.col[0] = reinterpret_cast<double*>(p);
    p += sizeof(double) * (cap + 4);
    sm.col[1] = reinterpret_cast<double*>(p);
    p += sizeof(double) * (cap + 4);
    sm.redd = reinterpret_cast<double*>(p);
    p += sizeof(double) * 32;
    sm.aug = reinterpret_cast<int*>(p);
    p += sizeof(int) * cap;
    sm.skip = reinterpret_cast<int*>(p);
    p += sizeof(int) * cap;
    sm.erow = reinterpret_cast<float*>(p);
    p += sizeof(float) * cap;
    sm.occ = reinterpret_cast<float*>(p);
    p += sizeof(float) * (cap / 2 + 2);
    sm.redf = reinterpret_cast<float*>(p);
    p += sizeof(float) * 64;
    sm.slot_of = reinterpret_cast<short*>(p);
  }
  for (int i = tid; i < cap + 4; i += NT) {
    sm.col[0][i] = NEG;
    sm.col[1][i] = NEG;
  }
  for (int s = tid; s < S; s += NT) sm.aug[s] = (s & 1) ? a.labels[u.lab_off + (s >> 1)] : a.blank;
  if (fused)
    for (int c = tid; c < a.A; c += NT) sm.slot_of[c] = -1;
  __syncthreads();
  for (int s = tid; s < S; s += NT)
    sm.skip[s] = (s >= 2 && sm.aug[s] != a.blank && sm.aug[s] != sm.aug[s - 2]) ? 1 : 0;
  if (fused)
    for (int j = tid; j < u.nkey; j += NT) sm.slot_of[a.key_char[u.key_off + j]] = static_cast<short>(j);
  __syncthreads();

  const size_t rs = static_cast<size_t>(a.B) * a.A;  // frame stride of [T][B][A]
  const float* xb = a.x + static_cast<size_t>(b) * a.A;
  double* st = a.store + u.store_off;  // column t at st + t*S; alpha(tm) at column T
  const int kmid = dir == 0 ? tm : T - 1 - tm;
  const int kgrad0 = dir == 0 ? tm : T - tm;

  int cell[K];
  bool live[K];
  float ex[K];        // prefetched raw logit of the next frame for each cell
  double cur[K];      // this CTA's lattice value of the current frame (alpha, or emission-exclusive beta)
  double other[K];    // the partner's stored value for the current gradient row
  double onext[K];    // ... prefetched for the next gradient row
#pragma unroll
  for (int j = 0; j < K; ++j) {
    cell[j] = tid + j * NT;
    live[j] = cell[j] < S;
    const int t0 = dir == 0 ? 0 : T - 1;
    ex[j] = live[j] ? __ldg(xb + static_cast<size_t>(t0) * rs + sm.aug[cell[j]]) : 0.f;
    other[j] = NEG;
    onext[j] = NEG;
  }
  // Fused gradient epilogue operands of the next gradient row (thread c owns symbol c; A <= NT).
  float xr_next = 0.f;
  float2 sts_next = make_float2(0.f, 0.f);
  if (fused && kgrad0 == 0 && tid < a.A) {  // forward CTA with T <= 2: row 0 is its first gradient row
    xr_next = __ldg(xb + tid);
    sts_next = a.stats[b];
  }
  double logz2 = 0.0;
  bool dead = false;  // log Z == -inf: zero-probability lattice (ctc.cpp:189-193)

  for (int k = 0; k < T; ++k) {
    const int t = dir == 0 ? k : T - 1 - k;
    double e[K];
#pragma unroll
    for (int j = 0; j < K; ++j) e[j] = static_cast<double>(ex[j]) * kLog2e;
    const float xr_cur = xr_next;
    const float2 sts_cur = sts_next;
    if (want_grad && k > kmid) {
#pragma unroll
      for (int j = 0; j < K; ++j) other[j] = onext[j];
    }
    if (k + 1 < T) {
      const int tn = dir == 0 ? k + 1 : T - 2 - k;
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (live[j]) ex[j] = __ldg(xb + static_cast<size_t>(tn) * rs + sm.aug[cell[j]]);
      if (fused && k + 1 >= kgrad0 && tid < a.A) {
        xr_next = __ldg(xb + static_cast<size_t>(tn) * rs + tid);
        sts_next = a.stats[static_cast<size_t>(tn) * a.B + b];
      }
    }

    // ---- one lattice column (ctc.cpp:109-124 forward / 126-143 backward) ----
    const double* colp = sm.col[(k + 1) & 1];
    double* colq = sm.col[k & 1];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (!live[j]) continue;
      const int s = cell[j];
      double v;
      if (dir == 0) {
        if (k == 0) {
          v = s < 2 ? e[j] : NEG;
        } else {
          v = lse3(colp[s + 2], colp[s + 1], sm.skip[s] ? colp[s] : NEG);
          v = v == NEG ? v : v + e[j];
        }
        colq[s + 2] = v;
      } else {
        if (k == 0) {
          v = s >= S - 2 ? 0.0 : NEG;
        } else {
          v = lse3(colp[s + 2], colp[s + 3], (s + 2 < S && sm.skip[s + 2]) ? colp[s + 4] : NEG);
        }
        colq[s + 2] = v == NEG ? v : v + e[j];  // emission-inclusive beta for the neighbours
      }
      cur[j] = v;
      if (k <= kmid) {
        const int col = (dir == 0 && k == tm) ? T : t;
        st[static_cast<size_t>(col) * S + s] = v;
      }
    }

    if (k == kmid) {
      // ---- meet in the middle: log Z = LSE_s alpha(s,tm) + beta(s,tm) ----
      __syncthreads();
      cluster_barrier();
      double vv[K];
      double mloc = NEG;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        vv[j] = NEG;
        if (!live[j]) continue;
        const int s = cell[j];
        const double o = st[static_cast<size_t>(dir == 0 ? tm : T) * S + s];
        if (dir == 0) other[j] = o;  // beta(tm): the forward CTA's first gradient row
        vv[j] = (o == NEG || cur[j] == NEG) ? NEG : cur[j] + o;
        mloc = vv[j] > mloc ? vv[j] : mloc;
      }
      mloc = warp_max_d(mloc);
      if (lane == 0) sm.redd[warp] = mloc;
      __syncthreads();
      double M = NEG;
      for (int w = 0; w < NW; ++w) M = sm.redd[w] > M ? sm.redd[w] : M;
      __syncthreads();
      if (M == NEG) {
        logz2 = NEG;
      } else {
        float sl = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) sl += ex2_approx(static_cast<float>(vv[j] - M));
        sl = warp_sum_f(sl);
        if (lane == 0) sm.redd[warp] = static_cast<double>(sl);
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < NW; ++w) tot += sm.redd[w];
        logz2 = M + log2(tot);
        __syncthreads();
      }
      dead = logz2 == NEG;
      if (!want_grad || dead) break;
    }
    // Prefetch the partner's stored column for the next gradient row (only
    // after the cluster barrier made it visible).
    if (want_grad && k >= kmid && k + 1 < T && k + 1 >= kgrad0) {
      const int tn = dir == 0 ? k + 1 : T - 2 - k;
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (live[j]) onext[j] = st[static_cast<size_t>(tn) * S + cell[j]];
    }

    if (want_grad && k >= kgrad0) {
      // ---- gradient row t (ctc.cpp:196-203, 69-79) ----
      float part = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (!live[j]) continue;
        const int s = cell[j];
        // gamma = alpha + beta as a PLAIN add (ctc.cpp:200): garbage + -inf cancels to -inf.
        const double g = cur[j] + other[j] - logz2;
        const float occ_s = ex2_approx(static_cast<float>(g));
        sm.erow[s] = occ_s;
        if (!(s & 1)) part += occ_s;
      }
      part = warp_sum_f(part);
      float* redf = sm.redf + 32 * (k & 1);
      if (lane == 0) redf[warp] = part;
      __syncthreads();
      // Non-blank symbols (and odd rows labelled with the blank id): ascending-row sums.
      for (int j = tid; j < u.nkey; j += NT) {
        const int r0 = a.key_start[u.key_off + b + j];
        const int r1 = a.key_start[u.key_off + b + j + 1];
        float acc = 0.f;
        for (int r = r0; r < r1; ++r) acc += sm.erow[a.key_rows[u.row_off + r]];
        sm.occ[j] = acc;
      }
      __syncthreads();
      if (fused) {
        if (tid < a.A) {
          const int slot = sm.slot_of[tid];
          float o = 0.f;
          if (slot == 0) {
            for (int w = 0; w < NW; ++w) o += redf[w];
            o += sm.occ[0];
          } else if (slot > 0) {
            o = sm.occ[slot];
          }
          const float soft = expf((xr_cur - sts_cur.x) - sts_cur.y);
          a.grad[static_cast<size_t>(t) * rs + static_cast<size_t>(b) * a.A + tid] = soft - o;
        }
      } else {
        float* orow = a.occ + u.occ_off + static_cast<size_t>(t) * u.nkey;
        for (int j = tid; j < u.nkey; j += NT) {
          float o = sm.occ[j];
          if (j == 0)
            for (int w = 0; w < NW; ++w) o += redf[w];
          orow[j] = o;
        }
      }
    } else {
      __syncthreads();
    }
  }

  if (fused) {
    if (dead) zero_rows(a, b, dir == 0 ? tm : 0, dir == 0 ? T : tm);
    if (dir == 1) zero_rows(a, b, T, a.t_max);
  }
  if (dir == 0 && warp == 0) {
    // cost = sum_t lse_t - log Z (natural log); deterministic lane-strided sum.
    double acc = 0.0;
    for (int t = lane; t < T; t += 32) {
      const float2 v = a.stats[static_cast<size_t>(t) * a.B + b];
      acc += static_cast<double>(v.x) + static_cast<double>(v.y);
    }
    acc = warp_sum_d(acc);
    if (lane == 0) {
      a.logz[b] = logz2;
      a.costs[b] = dead ? INFINITY : static_cast<float>(acc - logz2 * kLn2);
    }
  }
}

// ---------------------------------------------------------------------------
// K4: large-alphabet gradient, one coalesced pass per row:
// g = softmax(x_t) - occupancy (ctc.cpp:69-79), occupancy scattered only to
// the <= L+1 label symbols of the utterance (the key map), not densely.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_dense_grad(ChainArgs a) {
  const int row = blockIdx.x;
  const int t = row / a.B;
  const int b = row - t * a.B;
  const UttDesc u = a.desc[b];
  float* g = a.grad + static_cast<size_t>(row) * a.A;
  const float* xr = a.x + static_cast<size_t>(row) * a.A;
  const bool live = u.status == 0 && t < u.T && a.logz[b] != dneg_inf();
  if (!live) {
    for (int c = threadIdx.x; c < a.A; c += blockDim.x) g[c] = 0.f;
    return;
  }
  const float2 sv = a.stats[row];
  for (int c = threadIdx.x; c < a.A; c += blockDim.x) g[c] = expf((__ldg(xr + c) - sv.x) - sv.y);
  __syncthreads();
  const float* o = a.occ + u.occ_off + static_cast<size_t>(t) * u.nkey;
  for (int j = threadIdx.x; j < u.nkey; j += blockDim.x) g[a.key_char[u.key_off + j]] -= o[j];
}

size_t chain_smem_bytes(int nthreads, int cells, int A) {
  const size_t cap = static_cast<size_t>(nthreads) * cells;
  return sizeof(double) * (2 * (cap + 4) + 32) + sizeof(int) * 2 * cap + sizeof(float) * cap +
         sizeof(float) * (cap / 2 + 2) + sizeof(float) * 64 + sizeof(short) * (A <= kFusedMaxAlphabet ? A : 0) + 16;
}

template <int K>
int launch_chain_k(const ChainArgs& a, void* stream) {
  const size_t smem = chain_smem_bytes(a.nthreads, K, a.A);
  cudaError_t err = cudaFuncSetAttribute(k_pair_chain<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  k_pair_chain<K><<<2 * a.B, a.nthreads, smem, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

}  // namespace

int launch_rowstats(const ChainArgs& a, void* stream) {
  const long long rows = static_cast<long long>(a.t_max) * a.B;
  if (rows == 0) return cudaSuccess;
  const int blocks = static_cast<int>((rows * 32 + 255) / 256);
  k_rowstats<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a.x, const_cast<float2*>(a.stats), a.desc,
                                                                    a.t_max, a.B, a.A);
  return cudaGetLastError();
}

int launch_chain(const ChainArgs& a, void* stream) {
  if (a.B == 0) return cudaSuccess;
  switch (a.cells) {
    case 1: return launch_chain_k<1>(a, stream);
    case 2: return launch_chain_k<2>(a, stream);
    case 3: return launch_chain_k<3>(a, stream);
    case 4: return launch_chain_k<4>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

int launch_dense(const ChainArgs& a, void* stream) {
  const long long rows = static_cast<long long>(a.t_max) * a.B;
  if (rows == 0 || a.grad == nullptr) return cudaSuccess;
  k_dense_grad<<<static_cast<unsigned>(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

}  // namespace ds2ctc
