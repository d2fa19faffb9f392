// lse_step.cu -- microbenchmark of one CTC lattice step on sm_100a (design
// evidence, not product code). Each thread owns a (blank, label) cell pair and
// gets one neighbour value per step by warp shuffle, as in the pair kernel.
// Variants of the log-sum-exp arithmetic:
//   0 fp64 carry, fp32 MUFU correction (F2F conversions)
//   1 double-float (hi,lo fp32) carry, unsorted (3 ex2 + lg2 for the label cell)
//   2 double-float carry, sorted (max excluded: 2 ex2 + lg2 label, 1 ex2 + lg2 blank)
//   3 plain fp32 (precision floor, not usable: lower bound on cost)
// Reports cycles per step (clock64 in the kernel) for W warps per CTA, one CTA
// per SM. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 lse_step.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

struct DF { float h, l; };

__device__ __forceinline__ DF two_sum(float a, float b) {
  float s = a + b; float bb = s - a; float e = (a - (s - bb)) + (b - bb); return {s, e};
}
__device__ __forceinline__ DF fast2(float a, float b) { float s = a + b; return {s, b - (s - a)}; }

// x + corr + e  (double-float)
__device__ __forceinline__ DF df_add3(DF m, float corr, DF e) {
  DF s = two_sum(m.h, e.h);
  float lo = s.l + m.l + e.l + corr;
  return fast2(s.h, lo);
}

__device__ __forceinline__ DF lse2_unsorted(DF a, DF b, DF e) {
  float M = fmaxf(a.h, b.h);
  float s = ex2((a.h - M) + a.l) + ex2((b.h - M) + b.l);
  return df_add3({M, 0.f}, lg2(s), e);
}
__device__ __forceinline__ DF lse3_unsorted(DF a, DF b, DF c, DF e) {
  float M = fmaxf(fmaxf(a.h, b.h), c.h);
  float s = ex2((a.h - M) + a.l) + ex2((b.h - M) + b.l) + ex2((c.h - M) + c.l);
  return df_add3({M, 0.f}, lg2(s), e);
}
__device__ __forceinline__ DF lse2_sorted(DF a, DF b, DF e) {
  bool p = a.h >= b.h;
  DF hi = p ? a : b, lo = p ? b : a;
  float d = (lo.h - hi.h) + (lo.l - hi.l);
  return df_add3(hi, lg2(1.f + ex2(d)), e);
}
__device__ __forceinline__ DF lse3_sorted(DF a, DF b, DF c, DF e) {
  bool p = a.h >= b.h;
  DF hi = p ? a : b, lo = p ? b : a;
  bool q = hi.h >= c.h;
  DF m = q ? hi : c, o = q ? c : hi;
  float d1 = (lo.h - m.h) + (lo.l - m.l), d2 = (o.h - m.h) + (o.l - m.l);
  return df_add3(m, lg2(1.f + ex2(d1) + ex2(d2)), e);
}

__device__ __forceinline__ double lse_d(double a, double b, double c) {
  double m = a > b ? a : b; m = m > c ? m : c;
  float s = ex2((float)(a - m)) + ex2((float)(b - m)) + ex2((float)(c - m));
  return m + (double)lg2(s);
}
__device__ __forceinline__ double lse_d2(double a, double b) {
  double m = a > b ? a : b;
  float s = ex2((float)(a - m)) + ex2((float)(b - m));
  return m + (double)lg2(s);
}

template <int V>
__global__ void k(int T, const float* em, float* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  float e0 = em[threadIdx.x & 63], e1 = em[(threadIdx.x + 7) & 63];
  long long t0 = clock64();
  if (V == 0) {
    double bl = -1.0 * lane, lb = -2.0 * lane, d0 = e0, d1 = e1;
    for (int t = 0; t < T; ++t) {
      double nb = __shfl_up_sync(0xffffffffu, lb, 1);
      double nbl = lse_d2(bl, nb) + d0;
      double nlb = lse_d(lb, bl, nb) + d1;
      bl = nbl; lb = nlb;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(bl + lb);
  } else if (V == 3) {
    float bl = -1.f * lane, lb = -2.f * lane;
    for (int t = 0; t < T; ++t) {
      float nb = __shfl_up_sync(0xffffffffu, lb, 1);
      float M = fmaxf(bl, nb);
      float nbl = M + lg2(ex2(bl - M) + ex2(nb - M)) + e0;
      float M3 = fmaxf(M, lb);
      float nlb = M3 + lg2(ex2(lb - M3) + ex2(bl - M3) + ex2(nb - M3)) + e1;
      bl = nbl; lb = nlb;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = bl + lb;
  } else {
    DF bl = {-1.f * lane, 0.f}, lb = {-2.f * lane, 0.f};
    DF E0 = {e0, e0 * 1e-8f}, E1 = {e1, e1 * 1e-8f};
    for (int t = 0; t < T; ++t) {
      DF nb;
      nb.h = __shfl_up_sync(0xffffffffu, lb.h, 1);
      nb.l = __shfl_up_sync(0xffffffffu, lb.l, 1);
      DF nbl, nlb;
      if (V == 1) { nbl = lse2_unsorted(bl, nb, E0); nlb = lse3_unsorted(lb, bl, nb, E1); }
      else { nbl = lse2_sorted(bl, nb, E0); nlb = lse3_sorted(lb, bl, nb, E1); }
      bl = nbl; lb = nlb;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = bl.h + lb.h + bl.l + lb.l;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// conversion / MUFU pipe throughput probes: N independent chains per thread
__global__ void k_f2f(int n, double* io, long long* cyc) {
  double a = io[threadIdx.x], b = a + 1, c = a + 2, d = a + 3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a = (double)(float)a * 1.0000001; b = (double)(float)b * 1.0000001;
    c = (double)(float)c * 1.0000001; d = (double)(float)d * 1.0000001;
  }
  long long t1 = clock64();
  io[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_mufu(int n, float* io, long long* cyc) {
  float a = io[threadIdx.x], b = a + 1, c = a + 2, d = a + 3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = ex2(a) * -0.5f; b = ex2(b) * -0.5f; c = ex2(c) * -0.5f; d = ex2(d) * -0.5f; }
  long long t1 = clock64();
  io[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int T = 2000;
  float* em; float* out; long long* cyc; double* dio; float* fio;
  cudaMalloc(&em, 64 * 4); cudaMemset(em, 0, 64 * 4);
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&dio, 148 * 1024 * 8); cudaMemset(dio, 0, 148 * 1024 * 8);
  cudaMalloc(&fio, 148 * 1024 * 4); cudaMemset(fio, 0, 148 * 1024 * 4);
  long long h[148];
  const char* names[] = {"fp64-carry", "df-unsorted", "df-sorted", "fp32-plain"};
  for (int v = 0; v < 4; ++v) {
    for (int w : {1, 2, 4, 5, 8, 12, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (v) {
          case 0: k<0><<<148, 32 * w>>>(T, em, out, cyc); break;
          case 1: k<1><<<148, 32 * w>>>(T, em, out, cyc); break;
          case 2: k<2><<<148, 32 * w>>>(T, em, out, cyc); break;
          case 3: k<3><<<148, 32 * w>>>(T, em, out, cyc); break;
        }
      }
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      printf("%-12s warps=%2d  cycles/step=%7.1f\n", names[v], w, avg / T);
    }
  }
  for (int w : {1, 4, 8, 16, 32}) {
    k_f2f<<<148, 32 * w>>>(1000, dio, cyc); k_f2f<<<148, 32 * w>>>(1000, dio, cyc);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("f2f pair x4  warps=%2d cycles/iter=%7.1f  (lanes*8 conv per iter per SM: %d)\n", w, h[0] / 1000.0, 32 * w * 8);
    k_mufu<<<148, 32 * w>>>(1000, fio, cyc); k_mufu<<<148, 32 * w>>>(1000, fio, cyc);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mufu x4      warps=%2d cycles/iter=%7.1f  (lanes*4 ex2 per iter per SM: %d)\n", w, h[0] / 1000.0, 32 * w * 4);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
