// ctc_pair.cu -- the alpha || beta pair kernel of the DS2 CTC loss (sm_100a).
//
// Reference semantics: asr::ctc::ctc_loss_reference (proj/src/ctc.cpp:171-207)
// per utterance, using the column-parallel lattice scheme of
// ctc_loss_parallel (ctc.cpp:209-325; paper §5.2): every cell of a column is
// computed, invalid cells hold -inf or finite garbage that cancels in the
// plain alpha+beta add (ctc.cpp:200).
//
// One 2-CTA cluster per utterance. CTA 0 runs the forward recursion
// (forward_column, ctc.cpp:109-124), CTA 1 the emission-exclusive backward
// recursion (backward_column, ctc.cpp:126-143). Each stores its first half of
// the lattice; they meet at frame tm = (T-1)/2 (cluster barrier), compute
// log Z = log2 sum_s 2^(alpha(s,tm) + beta(s,tm)) identically, and then each
// streams its second half into occupancies gamma = alpha + beta - log Z,
// reading the partner's stored half. The serial chain is T steps, not 2T.
//
// Numerics: the recursion runs on the RAW logits in
// log2 units (per-frame normalisation cancels in gamma, and log p = log Z -
// sum_t lse_t); carried values are double-float (hi, lo fp32) so rounding does
// not accumulate as ulp(|alpha|) per step; the log-sum-exp correction uses
// MUFU ex2/lg2. Stored half-lattice cells are fp32 deltas from a per-warp max.
//
// Thread layout. Chain thread i owns label pairs i*K .. i*K+K-1. In the
// forward CTA pair j is (blank 2j, label 2j+1); in the backward CTA it is
// (label 2j-1, blank 2j). Either way a pair needs exactly ONE value from the
// neighbouring pair per step, which arrives by warp shuffle, or, across warp
// boundaries, through a tagged shared-memory ring (no CTA barrier per step).
// A service warp stages logits (cp.async) and the partner's columns, computes
// the per-frame log-softmax statistics, and turns occupancy rows into
// gradient rows (softmax - occupancy, ctc.cpp:69-79) one epoch behind the
// chain. All warps meet at a CTA barrier every P steps (an epoch).
#include <cuda_runtime.h>

#include <cstdint>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

constexpr float kL2eH = 1.44269502162933349609375f;  // fp32(log2 e)
constexpr float kL2eL = 1.925963033500011e-08f;      // log2 e - kL2eH
constexpr float kLn2f = 0.693147180559945309f;
constexpr double kLn2 = 0.69314718055994530942;
constexpr float NEGF = -__builtin_huge_valf();

struct DF {
  float h, l;
};

__device__ __forceinline__ DF dneg() { return {NEGF, 0.f}; }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ DF two_sum(float a, float b) {
  const float s = a + b;
  const float bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}

__device__ __forceinline__ DF fast2(float a, float b) {
  const float s = a + b;
  return {s, b - (s - a)};
}

// x * log2(e) as a double-float (x is exact in fp32).
__device__ __forceinline__ float2 emis_df(float x) {
  const float h = x * kL2eH;
  const float l = fmaf(x, kL2eH, -h) + x * kL2eL;
  return x == NEGF ? make_float2(NEGF, 0.f) : make_float2(h, l);
}

// Sorted log-sum-exp: the largest operand (by hi part) is kept exactly as the
// double-float base and only the others go through MUFU ex2, so a 2-way LSE
// costs ex2 + lg2 and a 3-way one 2 ex2 + lg2 (log_sum_exp_guarded,
// ctc.hpp:30-35: -inf operands contribute 0). Result = base + c.
struct LSE {
  DF base;
  float c;
};

__device__ __forceinline__ LSE lse2(DF a, DF b) {
  const bool p = a.h >= b.h;
  const DF hi = p ? a : b, lo = p ? b : a;
  const float d = (lo.h - hi.h) + (lo.l - hi.l);
  return {hi, lg2(1.f + ex2(d))};
}

__device__ __forceinline__ LSE lse3(DF a, DF b, DF c) {
  const bool p = a.h >= b.h;
  const DF hi = p ? a : b, lo = p ? b : a;
  const bool q = hi.h >= c.h;
  const DF m = q ? hi : c, o = q ? c : hi;
  const float d1 = (lo.h - m.h) + (lo.l - m.l);
  const float d2 = (o.h - m.h) + (o.l - m.l);
  return {m, lg2((1.f + ex2(d1)) + ex2(d2))};
}

// base + c + emission, with the reference guard `acc == -inf ? -inf : acc + lp` (ctc.cpp:231).
__device__ __forceinline__ DF incl(LSE m, float2 e) {
  const DF s = two_sum(m.base.h, e.x);
  const DF r = fast2(s.h, ((s.l + m.base.l) + e.y) + m.c);
  return (m.base.h == NEGF || e.x == NEGF) ? dneg() : r;
}

__device__ __forceinline__ DF excl(LSE m) {
  const DF r = fast2(m.base.h, m.base.l + m.c);
  return m.base.h == NEGF ? dneg() : r;
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ float warp_max_redux(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Tagged warp-boundary handoff: (hi, lo) with the step's low 8 bits in the
// lo mantissa (a 2^-16 relative perturbation of lo, i.e. ~2^-40 of the value).
// Predicated store (no branch, so no reconvergence point on the critical path).
__device__ __forceinline__ void bnd_put(bool pred, unsigned long long* slot, DF v, int tag) {
  const unsigned lo = (__float_as_uint(v.l) & ~0xFFu) | (static_cast<unsigned>(tag) & 0xFFu);
  const unsigned long long u = (static_cast<unsigned long long>(__float_as_uint(v.h)) << 32) | lo;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.volatile.shared.u64 [%0], %1;\n\t}" ::"r"(
          smem_addr(slot)),
      "l"(u), "r"(static_cast<unsigned>(pred)));
}

// Warp-uniform poll: every lane reads the same slot (a broadcast), so the
// spin loop never diverges; the caller keeps the value for one lane only.
__device__ __forceinline__ DF bnd_get(const unsigned long long* slot, int tag) {
  unsigned long long u;
  do {
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(u) : "r"(smem_addr(slot)));
  } while ((u & 0xFFull) != (static_cast<unsigned long long>(tag) & 0xFFull));
  return {__uint_as_float(static_cast<unsigned>(u >> 32)), __uint_as_float(static_cast<unsigned>(u) & ~0xFFu)};
}

#ifdef DS2CTC_EPOCH_TIMING
// Debug build only (tools/epoch_timing): per-epoch clock64 of every warp of the
// first cluster, [cta][epoch][warp][start, end].
__device__ long long g_epoch_clock[2][128][33][2];
#endif

// One epoch: steps [k0, k1) of a phase.
struct Epoch {
  int k0, k1, phase;  // phase 0 = none
};

template <int K>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMaxThreads, 1) k_pair(PairArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Geometry& g = a.g;
  const int dir = static_cast<int>(cluster_rank());  // 0: alpha forward, 1: beta backward
  const int b = a.order[blockIdx.x >> 1];
  const UttDesc u = a.desc[b];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int NT = blockDim.x;
  const int NCW = g.nchain;
  const bool want_grad = a.grad != nullptr;
  const bool fused = g.fused != 0;
  const size_t rs = static_cast<size_t>(a.B) * a.A;  // frame stride of [T][B][A]

  auto zero_rows = [&](int lo, int hi) {
    for (int t = lo; t < hi; ++t) {
      float* gr = a.grad + static_cast<size_t>(t) * rs + static_cast<size_t>(b) * a.A;
      for (int c = tid; c < a.A; c += NT) gr[c] = 0.f;
    }
  };

  if (u.status != 0) {  // infeasible (ctc.cpp:173) or T == 0 with an empty label
    if (dir == 0 && tid == 0) {
      a.logz[b] = u.status == 2 ? 0.0 : -__builtin_huge_val();
      if (fused) a.costs[b] = u.status == 2 ? 0.f : __builtin_huge_valf();
    }
    if (fused && want_grad) zero_rows(dir == 0 ? 0 : a.t_max / 2, dir == 0 ? a.t_max / 2 : a.t_max);
    return;
  }

  const int T = u.T, L = u.L, S = u.S, tm = u.tm;
  const int P = g.P, RX = 4 * P, P2 = 2 * P;  // powers of two
  const int MX = RX - 1, M2 = P2 - 1;
  const int S4 = round_up(S, 4);
  const int cw = u.col_w;
  const int nw_u = chain_warps_for(L, K);  // chain warps this utterance uses
  const int SW = g.SW;
  const int nstage = fused ? a.A : u.nkey;
  const int kmid = dir == 0 ? tm : T - 1 - tm;
  const int k2s = dir == 0 ? kmid : kmid + 1;  // first phase-2 step (gradient rows)
  const int kcount = dir == 0 ? kmid : kmid - 1;  // steps whose frame this CTA adds to sum lse

  float* xraw = reinterpret_cast<float*>(smem + g.off_xraw);
  float2* emis = reinterpret_cast<float2*>(smem + g.off_emis);
  float2* lser = reinterpret_cast<float2*>(smem + g.off_lse);
  float* eb = reinterpret_cast<float*>(smem + g.off_eb);
  float* el = reinterpret_cast<float*>(smem + g.off_el);
  float* sring = reinterpret_cast<float*>(smem + g.off_sring);
  float* tile = reinterpret_cast<float*>(smem + g.off_tile);
  float* occs = reinterpret_cast<float*>(smem + g.off_occ);
  unsigned long long* bnd = reinterpret_cast<unsigned long long*>(smem + g.off_bnd);
  int* s_lab = reinterpret_cast<int*>(smem + g.off_meta);
  int* s_kchar = s_lab + (L + 1);
  int* s_kstart = s_kchar + u.nkey;
  int* s_kpos = s_kstart + u.nkey + 1;
  int* s_slotpos = s_kpos + L;  // slot of each label position
  short* s_slot = reinterpret_cast<short*>(s_slotpos + L + 1);  // fused: symbol -> slot
  double* red = reinterpret_cast<double*>(smem + g.off_red);

  // ---- prologue: per-utterance metadata into shared memory ----
  for (int i = tid; i < L; i += NT) s_lab[i] = a.labels[u.lab_off + i];
  for (int j = tid; j < u.nkey; j += NT) s_kchar[j] = a.key_char[u.key_off + j];
  for (int j = tid; j <= u.nkey; j += NT) s_kstart[j] = a.key_start[u.key_off + b + j];
  for (int q = tid; q < L; q += NT) s_kpos[q] = a.key_pos[u.lab_off + q];
  if (fused)
    for (int c = tid; c < a.A; c += NT) s_slot[c] = -1;
  for (int q = tid; q < NCW * P2; q += NT) bnd[q] = ~0ull;
  __syncthreads();
  if (fused)
    for (int j = tid; j < u.nkey; j += NT) s_slot[s_kchar[j]] = static_cast<short>(j);
  for (int j = tid; j < u.nkey; j += NT)
    for (int q = s_kstart[j]; q < s_kstart[j + 1]; ++q) s_slotpos[s_kpos[q]] = j;
  __syncthreads();

  auto frame = [&](int k) { return dir == 0 ? k : T - 1 - k; };
  auto next_epoch = [&](const Epoch& e) -> Epoch {
    if (e.phase == 1) {
      if (e.k1 <= kmid) return {e.k1, min(e.k1 + P, kmid + 1), 1};
      if (want_grad && k2s < T) return {k2s, min(k2s + P, T), 2};
      return {0, 0, 0};
    }
    if (e.phase == 2 && e.k1 < T) return {e.k1, min(e.k1 + P, T), 2};
    return {0, 0, 0};
  };

  // ---- per-thread chain state ----
  const bool is_chain = warp < nw_u;
  const bool service = warp == NCW;
  const int sidx_b = fused ? a.blank : 0;  // staged index of the blank symbol
  int sidx_l[K];                           // staged index of each pair's label symbol
  bool skip[K];                            // skip_allowed(2i+1) (ctc.cpp:41-43)
  bool has_b[K], has_l[K];
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const int i = tid * K + p;
    has_b[p] = is_chain && i <= L;
    const int li = dir == 0 ? i : i - 1;  // label index of this pair's label cell
    has_l[p] = is_chain && li >= 0 && li < L;
    const int sym = has_l[p] ? s_lab[li] : a.blank;
    sidx_l[p] = fused ? sym : (has_l[p] ? s_slotpos[li] : 0);
    skip[p] = is_chain && i >= 1 && i < L && s_lab[i] != a.blank && s_lab[i] != s_lab[i - 1];
  }
  DF vb[K], vl[K];  // published values: alpha (forward) or emission-inclusive beta~ (backward)
  DF xb[K], xl[K];  // backward only: emission-exclusive beta (storage / occupancy)
  DF qb[K], ql[K];  // the previous column's stored/occupancy values (aux work runs one step behind)
  float pwb[K], pdb[K], pwl[K], pdl[K];  // partner (woff, delta) of the row the aux step consumes
  float nwb[K], ndb[K], nwl[K], ndl[K];  // ... prefetched for the next row
#pragma unroll
  for (int p = 0; p < K; ++p) {
    vb[p] = vl[p] = xb[p] = xl[p] = qb[p] = ql[p] = dneg();
    pwb[p] = pdb[p] = pwl[p] = pdl[p] = nwb[p] = ndb[p] = nwl[p] = ndl[p] = NEGF;
  }
  float2 eBp[K], eL[K];  // emissions of the next column (blank, label) per pair
#pragma unroll
  for (int p = 0; p < K; ++p) eBp[p] = eL[p] = make_float2(0.f, 0.f);
  float wprev = NEGF;  // warp max of the previous column (CREDUX issued one step earlier)
  float Zh = 0.f, Zl = 0.f;
  double logz2 = 0.0;
  double lse_acc = 0.0;  // service warp lanes: sum of counted lse (natural log)

  // ---- service warp: staging / conversion / statistics ----
  auto stage = [&](const Epoch& e, bool partner) {
    if (e.phase == 0) return;
    for (int k = e.k0; k < e.k1; ++k) {
      const float* src = a.x + static_cast<size_t>(frame(k)) * rs + static_cast<size_t>(b) * a.A;
      float* dst = xraw + (k & MX) * g.xstride;
      for (int c = lane; c < nstage; c += 32) cp_async4(dst + c, src + (fused ? c : s_kchar[c]));
      if (partner && e.phase == 2) {
        const float* col = a.store + u.store_off + static_cast<size_t>(frame(k)) * cw;
        float* sdst = sring + (k & M2) * g.cw_max;
        for (int c4 = lane; c4 < cw / 4; c4 += 32) cp_async16(sdst + 4 * c4, col + 4 * c4);
      }
    }
    cp_async_commit();
  };
  auto convert = [&](const Epoch& e) {  // after the staged data landed (wait + __syncwarp)
    if (e.phase == 0) return;
    const int n = e.k1 - e.k0;
    for (int k = e.k0; k < e.k1; ++k)
      for (int c = lane; c < nstage; c += 32) emis[(k & M2) * SW + c] = emis_df(xraw[(k & MX) * g.xstride + c]);
    if (fused && lane < n) {  // per-frame (max, log sum exp), lane = frame (ctc.cpp:24-37)
      const int k = e.k0 + lane;
      const float* xr = xraw + (k & MX) * g.xstride;
      float m0 = NEGF, m1 = NEGF;
      int c = 0;
      for (; c + 1 < a.A; c += 2) {
        m0 = fmaxf(m0, xr[c]);
        m1 = fmaxf(m1, xr[c + 1]);
      }
      if (c < a.A) m0 = fmaxf(m0, xr[c]);
      const float m = fmaxf(m0, m1);
      float s0 = 0.f, s1 = 0.f;
      for (c = 0; c + 1 < a.A; c += 2) {
        s0 += ex2((xr[c] - m) * kL2eH);
        s1 += ex2((xr[c + 1] - m) * kL2eH);
      }
      if (c < a.A) s0 += ex2((xr[c] - m) * kL2eH);
      const float ls = lg2(s0 + s1) * kLn2f;
      lser[k & MX] = make_float2(m, ls);
      if (k <= kcount) lse_acc += static_cast<double>(m) + static_cast<double>(ls);
    }
  };
  // Gradient rows of a finished phase-2 epoch, lane = row (ctc.cpp:196-203, 69-79).
  auto grad_rows = [&](const Epoch& e) {
    if (e.phase != 2) return;
    const int n = e.k1 - e.k0;
    if (lane < n) {
      const int k = e.k0 + lane;
      const float* ebr = eb + (k & M2) * g.estride;
      const float* elr = el + (k & M2) * g.estride;
      float* oc = occs + lane * g.ostride;
      float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;  // blank rows (every even lattice row), fixed order
      int i = 0;
      for (; i + 3 <= L; i += 4) {
        b0 += ebr[i];
        b1 += ebr[i + 1];
        b2 += ebr[i + 2];
        b3 += ebr[i + 3];
      }
      for (; i <= L; ++i) b0 += ebr[i];
      const float bsum = (b0 + b1) + (b2 + b3);
      for (int j = 0; j < u.nkey; ++j) {
        const int q0 = s_kstart[j], q1 = s_kstart[j + 1];
        float a0 = j == 0 ? bsum : 0.f, a1 = 0.f;
        int q = q0;
        for (; q + 1 < q1; q += 2) {
          a0 += elr[s_kpos[q]];
          a1 += elr[s_kpos[q + 1]];
        }
        if (q < q1) a0 += elr[s_kpos[q]];
        oc[j] = a0 + a1;
      }
      float* tr = tile + lane * g.tstride;
      if (fused) {
        const float2 st = lser[k & MX];
        const float* xr = xraw + (k & MX) * g.xstride;
#pragma unroll 4
        for (int c = 0; c < a.A; ++c) {
          const int slot = s_slot[c];
          const float soft = ex2(((xr[c] - st.x) - st.y) * kL2eH);
          tr[c] = soft - (slot >= 0 ? oc[slot] : 0.f);
        }
      } else {
        for (int j = 0; j < u.nkey; ++j) tr[j] = oc[j];
      }
    }
    __syncwarp();
    for (int r = 0; r < n; ++r) {
      const int t = frame(e.k0 + r);
      const float* tr = tile + r * g.tstride;
      if (fused) {
        float* gr = a.grad + static_cast<size_t>(t) * rs + static_cast<size_t>(b) * a.A;
        for (int c = lane; c < a.A; c += 32) gr[c] = tr[c];
      } else {
        float* orow = a.occ + u.occ_off + static_cast<size_t>(t) * u.nkey;
        for (int j = lane; j < u.nkey; j += 32) orow[j] = tr[j];
      }
    }
    __syncwarp();
  };

  // ---- chain: critical part of step k (one lattice column) ----
  // Cells that do not exist get a -inf emission, which makes incl() return
  // -inf without a predicate on the critical path.
  auto load_emis = [&](int k) {
    const float2* er = emis + (k & M2) * SW;
    const float2 ninf = make_float2(NEGF, 0.f);
    const float2 e0 = er[sidx_b];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      eBp[p] = has_b[p] ? e0 : ninf;
      const float2 e1 = er[sidx_l[p]];
      eL[p] = has_l[p] ? e1 : ninf;
    }
  };
  auto first_column = [&]() {
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int i = tid * K + p;
      if (dir == 0) {  // alpha(s, 0) = lp(0, aug[s]) for s < 2 (ctc.cpp:114)
        vb[p] = i == 0 ? DF{eBp[p].x, eBp[p].y} : dneg();
        vl[p] = i == 0 ? DF{eL[p].x, eL[p].y} : dneg();
        if (eBp[p].x == NEGF) vb[p] = dneg();
        if (eL[p].x == NEGF) vl[p] = dneg();
      } else {  // beta(s, T-1) = 0 for s >= S-2 (ctc.cpp:130)
        const bool last = i == L;
        const LSE zero{{0.f, 0.f}, 0.f};
        xb[p] = (last && has_b[p]) ? DF{0.f, 0.f} : dneg();
        xl[p] = (last && has_l[p]) ? DF{0.f, 0.f} : dneg();
        vb[p] = last ? incl(zero, eBp[p]) : dneg();
        vl[p] = last ? incl(zero, eL[p]) : dneg();
      }
    }
    if (dir == 0) bnd_put(lane == 31 && warp + 1 < nw_u, bnd + warp * P2, vl[K - 1], 0);
    else bnd_put(lane == 0 && warp > 0, bnd + warp * P2, vl[0], 0);
  };
  auto critical = [&](int k) {  // k >= 1; branch-free except the warp-uniform poll
    if (dir == 0) {
      DF nb;
      nb.h = __shfl_up_sync(0xffffffffu, vl[K - 1].h, 1);
      nb.l = __shfl_up_sync(0xffffffffu, vl[K - 1].l, 1);
      if (warp > 0) {
        const DF bv = bnd_get(bnd + (warp - 1) * P2 + ((k - 1) & M2), k - 1);
        if (lane == 0) nb = bv;
      } else if (lane == 0) {
        nb = dneg();
      }
      DF nvb[K], nvl[K];
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const DF n1 = p == 0 ? nb : vl[p - 1];
        const LSE mb = lse2(vb[p], n1);                            // blank 2i <- 2i, 2i-1
        const LSE ml = lse3(vl[p], vb[p], skip[p] ? n1 : dneg());  // label 2i+1 <- 2i+1, 2i, 2i-1
        nvb[p] = incl(mb, eBp[p]);
        nvl[p] = incl(ml, eL[p]);
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        vb[p] = nvb[p];
        vl[p] = nvl[p];
      }
      bnd_put(lane == 31 && warp + 1 < nw_u, bnd + warp * P2 + (k & M2), vl[K - 1], k);
    } else {
      DF nb;
      nb.h = __shfl_down_sync(0xffffffffu, vl[0].h, 1);
      nb.l = __shfl_down_sync(0xffffffffu, vl[0].l, 1);
      if (warp + 1 < nw_u) {
        const DF bv = bnd_get(bnd + (warp + 1) * P2 + ((k - 1) & M2), k - 1);
        if (lane == 31) nb = bv;
      } else if (lane == 31) {
        nb = dneg();
      }
      DF nvb[K], nvl[K];
#pragma unroll
      for (int p = K - 1; p >= 0; --p) {
        const DF n1 = p == K - 1 ? nb : vl[p + 1];
        const LSE mb = lse2(vb[p], n1);                            // blank 2i <- 2i, 2i+1
        const LSE ml = lse3(vl[p], vb[p], skip[p] ? n1 : dneg());  // label 2i-1 <- 2i-1, 2i, 2i+1
        nvb[p] = incl(mb, eBp[p]);
        nvl[p] = incl(ml, eL[p]);
        xb[p] = excl(mb);  // only stored / used where the cell exists
        xl[p] = excl(ml);
      }
#pragma unroll
      for (int p = 0; p < K; ++p) {
        vb[p] = nvb[p];
        vl[p] = nvl[p];
      }
      bnd_put(lane == 0 && warp > 0, bnd + warp * P2 + (k & M2), vl[0], k);
    }
  };
  // Values of the current column that storage / occupancy use (alpha, or emission-exclusive beta).
  auto snapshot = [&]() {
#pragma unroll
    for (int p = 0; p < K; ++p) {
      qb[p] = dir == 0 ? vb[p] : xb[p];
      ql[p] = dir == 0 ? vl[p] : xl[p];
    }
  };
  auto column_max = [&]() {  // warp max of the hi parts of the snapshot (CREDUX)
    float hm = NEGF;
#pragma unroll
    for (int p = 0; p < K; ++p) hm = fmaxf(hm, fmaxf(qb[p].h, ql[p].h));
    return warp_max_redux(hm);
  };
  // Phase-1 column store of the snapshot: fp32 delta from the warp max of the hi parts.
  auto store_column = [&](int k, float wmax) {
    const int col = (dir == 0 && k == kmid) ? T : frame(k);
    float* dst = a.store + u.store_off + static_cast<size_t>(col) * cw;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int i = tid * K + p;
      const float db = qb[p].h == NEGF ? NEGF : (qb[p].h - wmax) + qb[p].l;
      const float dl = ql[p].h == NEGF ? NEGF : (ql[p].h - wmax) + ql[p].l;
      if (has_b[p]) dst[2 * i] = db;
      if (has_l[p]) dst[dir == 0 ? 2 * i + 1 : 2 * i - 1] = dl;
    }
    if (lane == 0) dst[S4 + warp] = wmax;
  };
  // Partner (woff, delta) of each of my cells for row k (the partner's stored column).
  auto load_partner = [&](int k) {
    const float* col = sring + (k & M2) * g.cw_max;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int i = tid * K + p;
      const int sb = 2 * i, sl = dir == 0 ? 2 * i + 1 : 2 * i - 1;
      const int wb = dir == 0 ? (sb + 1) / (64 * K) : sb / (64 * K);  // partner's writer warp
      const int wl = dir == 0 ? (sl + 1) / (64 * K) : sl / (64 * K);
      nwb[p] = has_b[p] ? col[S4 + wb] : NEGF;
      ndb[p] = has_b[p] ? col[sb] : NEGF;
      nwl[p] = has_l[p] ? col[S4 + wl] : NEGF;
      ndl[p] = has_l[p] ? col[sl] : NEGF;
    }
  };
  // gamma = alpha + beta - log Z (plain add, ctc.cpp:200) -> occupancy 2^gamma.
  auto occupancy = [&](DF v, float woff, float delta) -> float {
    const DF p = two_sum(v.h, -Zh);
    const float q = p.h + woff;
    const float gg = q + ((p.l + v.l) + (delta - Zl));
    const float o = ex2(gg);
    return (v.h == NEGF || woff == NEGF || delta == NEGF) ? 0.f : o;
  };
  auto occupancy_row = [&](int k) {  // uses the snapshot and pw*/pd*
    float* ebr = eb + (k & M2) * g.estride;
    float* elr = el + (k & M2) * g.estride;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const int i = tid * K + p;
      if (has_b[p]) ebr[i] = occupancy(qb[p], pwb[p], pdb[p]);
      if (has_l[p]) elr[dir == 0 ? i : i - 1] = occupancy(ql[p], pwl[p], pdl[p]);
    }
  };

  // One epoch of chain work. The critical recursion of step k is issued
  // first; the column store (phase 1) or occupancy row (phase 2) of step k-1
  // follows, so its latency overlaps the next column instead of stalling it.
  auto chain_epoch = [&](const Epoch& e) {
    load_emis(e.k0);
    for (int k = e.k0; k < e.k1; ++k) {
      if (k == 0) first_column();
      else if (e.phase == 1 || k > kmid) critical(k);
#ifndef DS2CTC_EXP_NOEMIS
      if (k + 1 < e.k1) load_emis(k + 1);
#endif
      if (e.phase == 1) {
#ifndef DS2CTC_EXP_NOSTORE
        const float wnow = [&] {
          // snapshot of column k taken after the previous column was stored
          if (k > e.k0) store_column(k - 1, wprev);
          snapshot();
#ifdef DS2CTC_EXP_NOREDUX
          return 0.f;
#else
          return column_max();
#endif
        }();
        wprev = wnow;
#endif
      } else {
        load_partner(k);
        if (k > e.k0) occupancy_row(k - 1);
        snapshot();
#pragma unroll
        for (int p = 0; p < K; ++p) {
          pwb[p] = nwb[p];
          pdb[p] = ndb[p];
          pwl[p] = nwl[p];
          pdl[p] = ndl[p];
        }
      }
    }
    if (e.phase == 1) {
      store_column(e.k1 - 1, wprev);
    } else {
      occupancy_row(e.k1 - 1);
    }
  };

  // ---- prologue staging of epoch 0 ----
  Epoch cur{0, min(P, kmid + 1), 1};
  if (service) {
    stage(cur, false);
    cp_async_wait_all();
    __syncwarp();
    convert(cur);
  }
  __syncthreads();

  Epoch prev{0, 0, 0};
  bool dead = false;
#ifdef DS2CTC_EPOCH_TIMING
  int epoch_idx = 0;
#endif
  while (cur.phase != 0) {
    const Epoch nxt = next_epoch(cur);
#ifdef DS2CTC_EPOCH_TIMING
    if (blockIdx.x < 2 && lane == 0 && epoch_idx < 128) g_epoch_clock[dir][epoch_idx][warp][0] = clock64();
#endif
    // The forward CTA's first phase-2 epoch starts at kmid, which the last
    // phase-1 epoch already staged: stage only steps not staged yet.
    Epoch stg = nxt;
    if (stg.phase != 0 && stg.k0 < cur.k1) stg.k0 = cur.k1;
    if (service) {
      stage(stg, cur.phase == 2);
      grad_rows(prev);
      cp_async_wait_all();
      __syncwarp();
      convert(stg);
    } else if (is_chain) {
      chain_epoch(cur);
    }
#ifdef DS2CTC_EPOCH_TIMING
    if (blockIdx.x < 2 && lane == 0 && epoch_idx < 128) g_epoch_clock[dir][epoch_idx][warp][1] = clock64();
    ++epoch_idx;
#endif
    __syncthreads();
    if (cur.phase == 1 && cur.k1 == kmid + 1) {
      // ---- meet in the middle: log Z (all threads of both CTAs) ----
      cluster_barrier();
      // Both CTAs read the two STORED columns (alpha(tm) at column T, beta(tm)
      // at column tm) with the same cell->thread map and reduction order, so
      // they derive the bitwise-identical log Z.
      const float* ca = a.store + u.store_off + static_cast<size_t>(T) * cw;
      const float* cb = a.store + u.store_off + static_cast<size_t>(tm) * cw;
      double mloc = -__builtin_huge_val();
      for (int s = tid; s < S; s += NT) {
        const float wa = ca[S4 + s / (64 * K)], da = ca[s];
        const float wb = cb[S4 + (s + 1) / (64 * K)], db = cb[s];
        if (wa == NEGF || da == NEGF || wb == NEGF || db == NEGF) continue;
        const double v = (static_cast<double>(wa) + static_cast<double>(da)) +
                         (static_cast<double>(wb) + static_cast<double>(db));
        mloc = v > mloc ? v : mloc;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, mloc, o);
        mloc = w > mloc ? w : mloc;
      }
      if (lane == 0) red[warp] = mloc;
      __syncthreads();
      double M = -__builtin_huge_val();
      for (int w = 0; w < NT / 32; ++w) M = red[w] > M ? red[w] : M;
      if (M == -__builtin_huge_val()) {
        logz2 = M;
      } else {
        float sl = 0.f;
        for (int s = tid; s < S; s += NT) {
          const float wa = ca[S4 + s / (64 * K)], da = ca[s];
          const float wb = cb[S4 + (s + 1) / (64 * K)], db = cb[s];
          if (wa == NEGF || da == NEGF || wb == NEGF || db == NEGF) continue;
          const double v = (static_cast<double>(wa) + static_cast<double>(da)) +
                           (static_cast<double>(wb) + static_cast<double>(db));
          sl += ex2(static_cast<float>(v - M));
        }
        for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
        if (lane == 0) red[32 + warp] = static_cast<double>(sl);
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < NT / 32; ++w) tot += red[32 + w];
        logz2 = M + log2(tot);
      }
      Zh = static_cast<float>(logz2);
      Zl = static_cast<float>(logz2 - static_cast<double>(Zh));
      dead = logz2 == -__builtin_huge_val();  // zero-probability lattice (ctc.cpp:189-193)
      if (dead || !want_grad) break;
      // Partner columns of the first phase-2 epoch (now visible after the cluster barrier).
      if (service) {
        const Epoch first = next_epoch(cur);
        for (int k = first.k0; k < first.k1; ++k) {
          const float* col = a.store + u.store_off + static_cast<size_t>(frame(k)) * cw;
          for (int c4 = lane; c4 < cw / 4; c4 += 32) cp_async16(sring + (k & M2) * g.cw_max + 4 * c4, col + 4 * c4);
        }
        cp_async_commit();
        cp_async_wait_all();
      }
      __syncthreads();
    }
    prev = cur;
    cur = nxt;
  }
  if (service && !dead && want_grad) grad_rows(prev);  // the last phase-2 epoch

  // ---- costs: cost = sum_t lse_t - log Z (natural log) ----
  if (fused) {
    if (want_grad) {
      if (dead) zero_rows(dir == 0 ? tm : 0, dir == 0 ? T : tm);
      if (dir == 1) zero_rows(T, a.t_max);
    }
    if (service) {
      for (int o = 16; o > 0; o >>= 1) lse_acc += __shfl_xor_sync(0xffffffffu, lse_acc, o);
      if (lane == 0) a.part[2 * b + dir] = lse_acc;
    }
    cluster_barrier();
    if (dir == 0 && tid == 0) {
      const double tot = a.part[2 * b] + a.part[2 * b + 1];
      a.logz[b] = logz2;
      a.costs[b] = dead ? __builtin_huge_valf() : static_cast<float>(tot - logz2 * kLn2);
    }
  } else if (dir == 0 && tid == 0) {
    a.logz[b] = logz2;
  }
}

template <int K>
int launch_k(const PairArgs& a, void* stream) {
  const int threads = 32 * (a.g.nchain + 1);
  if (threads > kMaxThreads) return cudaErrorInvalidValue;
  cudaError_t err = cudaFuncSetAttribute(k_pair<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, a.g.smem);
  if (err != cudaSuccess) return err;
  k_pair<K><<<2 * a.B, threads, a.g.smem, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError();
}

}  // namespace

#ifdef DS2CTC_EPOCH_TIMING
extern "C" int ds2ctc_debug_epoch_clocks(long long* host) {
  return cudaMemcpyFromSymbol(host, g_epoch_clock, sizeof(g_epoch_clock));
}
#endif

int launch_pair(const PairArgs& a, void* stream) {
  if (a.B == 0) return cudaSuccess;
  switch (a.g.K) {
    case 1: return launch_k<1>(a, stream);
    case 2: return launch_k<2>(a, stream);
    case 3: return launch_k<3>(a, stream);
    case 4: return launch_k<4>(a, stream);
    case 6: return launch_k<6>(a, stream);
    case 8: return launch_k<8>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ds2ctc
