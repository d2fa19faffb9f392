// chain_step.cu -- microbenchmark of one chain warp's lattice step (design
// evidence, not product code): K label pairs per lane, emissions from a shared
// ring (warp-uniform row), neighbour by shuffle, per-thread offset re-centring,
// column stores to shared memory. One warp per SM sub-partition (4 per CTA,
// independent), 148 CTAs. Variants:
//   V=0 lse2 + lse3 (the product kernel's arithmetic, 5 MUFU per pair)
//   V=1 lse2 + lse2 (label cell = lse2(label, skip ? blank_lse : blank), 4 MUFU)
//   V=2 as 1, re-centring shift lagged by one step (applied with the emission)
//   V=3 linear-in-step: one ex2 per cell, sums in linear, one lg2 per cell (4 MUFU per pair + 1)
//   V=4 as 3 + a per-step fragility vote (any live cell below -100 -> exact step)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 chain_step.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lse2(float a, float b) { return fmaxf(a, b) + lg2(1.f + ex2(-fabsf(a - b))); }
__device__ __forceinline__ float lse3(float a, float b, float c) {
  const float hi = fmaxf(a, b), d1 = a - b, d2 = hi - c;
  return fmaxf(hi, c) + lg2((1.f + ex2(fminf(d2, 0.f) - fabsf(d1))) + ex2(-fabsf(d2)));
}
constexpr float SENT = -1e30f;

template <int K, int V>
__global__ void __launch_bounds__(128, 1) kstep(int T, float* out, long long* cyc) {
  __shared__ float emis[64 * 33];
  __shared__ __align__(16) float cb[4][4][2 * K * 32 + 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 33; i += blockDim.x) emis[i] = -1.f - (float)((i * 7919) % 97) * 0.05f;
  __syncthreads();
  unsigned ea_l[K];
  bool skip[K];
  float vb[K], vl[K];
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const int sym = ((lane * K + p) * 7) % 29;
    ea_l[p] = (unsigned)__cvta_generic_to_shared(emis + sym);
    skip[p] = ((lane + p) % 5) != 0;
    vb[p] = -0.5f * p;
    vl[p] = -0.25f * p;
  }
  const unsigned ea_b = (unsigned)__cvta_generic_to_shared(emis + 28);
  float O = 0.f, shp = 0.f;
  float* colbase = &cb[warp][0][2 * K * lane];
  long long t0 = clock64();
#pragma unroll 1
  for (int t = 1; t < T; ++t) {
    const unsigned row = (unsigned)((t & 63) * 33 * 4);
    float eb, el[K];
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(eb) : "r"(ea_b + row));
#pragma unroll
    for (int p = 0; p < K; ++p) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(el[p]) : "r"(ea_l[p] + row));
    float nr = __shfl_up_sync(0xffffffffu, vl[K - 1], 1);
    float no = __shfl_up_sync(0xffffffffu, O, 1);
    nr = lane == 0 ? SENT : nr;
    no = lane == 0 ? O : no;
    const float n0 = nr + (no - O);
    float nvb[K], nvl[K];
    if (V >= 2) {
      eb -= shp;
#pragma unroll
      for (int p = 0; p < K; ++p) el[p] -= shp;
    }
    if (V >= 3) {
      float Eb[K], El[K];
#pragma unroll
      for (int p = 0; p < K; ++p) { Eb[p] = ex2(vb[p]); El[p] = ex2(vl[p]); }
      const float En = ex2(n0);
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const float n1 = p == 0 ? En : El[p - 1];
        nvb[p] = lg2(Eb[p] + n1) + eb;
        nvl[p] = lg2(fmaf(skip[p] ? 1.f : 0.f, n1, El[p]) + Eb[p]) + el[p];
      }
    } else
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const float n1 = p == 0 ? n0 : vl[p - 1];
      const float mb = lse2(vb[p], n1);
      float ml;
      if (V == 0) ml = lse3(vl[p], vb[p], skip[p] ? n1 : SENT);
      else ml = lse2(vl[p], skip[p] ? mb : vb[p]);
      nvb[p] = mb + eb;
      nvl[p] = ml + el[p];
    }
    float mx = fmaxf(nvb[0], nvl[0]);
#pragma unroll
    for (int p = 1; p < K; ++p) mx = fmaxf(mx, fmaxf(nvb[p], nvl[p]));
    const float sh = __fsub_rn(__fadd_rn(mx, 12582912.f), 12582912.f);
    if (V == 4) {
      bool frag = n0 < -100.f && n0 > -1e29f;
#pragma unroll
      for (int p = 0; p < K; ++p) frag |= (nvb[p] - mx < -100.f && nvb[p] > -1e29f) | (nvl[p] - mx < -100.f && nvl[p] > -1e29f);
      if (__any_sync(0xffffffffu, frag)) O += 1.f;  // stand-in for the exact step
    }
    if (V >= 2) {
#pragma unroll
      for (int p = 0; p < K; ++p) { vb[p] = nvb[p]; vl[p] = nvl[p]; }
      O += shp;
      shp = sh;
    } else {
#pragma unroll
      for (int p = 0; p < K; ++p) { vb[p] = nvb[p] - sh; vl[p] = nvl[p] - sh; }
      O += sh;
    }
    float* dst = colbase + (t & 3) * (2 * K * 32 + 4);
#pragma unroll
    for (int p = 0; p < K; ++p) reinterpret_cast<float2*>(dst)[p] = make_float2(vb[p], vl[p]);
  }
  long long t1 = clock64();
  float s = O;
#pragma unroll
  for (int p = 0; p < K; ++p) s += vb[p] + vl[p];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + cb[warp][lane & 3][0];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K, int V>
void run(float* out, long long* cyc) {
  const int T = 4000;
  long long h[148];
  for (int rep = 0; rep < 2; ++rep) kstep<K, V><<<148, 128>>>(T, out, cyc);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("V=%d K=%d cycles/step=%7.1f\n", V, K, s / 148 / (T - 1));
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 128 * 4); cudaMalloc(&cyc, 148 * 8);
  run<2, 0>(out, cyc); run<3, 0>(out, cyc); run<4, 0>(out, cyc); run<5, 0>(out, cyc); run<6, 0>(out, cyc);
  run<2, 1>(out, cyc); run<3, 1>(out, cyc); run<4, 1>(out, cyc); run<5, 1>(out, cyc); run<6, 1>(out, cyc);
  run<2, 2>(out, cyc); run<3, 2>(out, cyc); run<4, 2>(out, cyc); run<5, 2>(out, cyc); run<6, 2>(out, cyc);
  run<2, 3>(out, cyc); run<3, 3>(out, cyc); run<4, 3>(out, cyc); run<5, 3>(out, cyc); run<6, 3>(out, cyc);
  run<2, 4>(out, cyc); run<3, 4>(out, cyc); run<4, 4>(out, cyc); run<5, 4>(out, cyc); run<6, 4>(out, cyc);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
