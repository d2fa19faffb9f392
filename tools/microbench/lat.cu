// lat.cu -- dependent-chain latency of the chain step's primitives on sm_100a
// (design evidence): FADD, FMNMX, MUFU.EX2, MUFU.LG2, SHFL, LDS, ex2+lg2 pair.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int V>
__global__ void k(int n, float* io, long long* cyc) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 0.f;
  __syncthreads();
  float a = io[threadIdx.x];
  unsigned u = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (V == 0) { asm volatile("add.f32 %0, %0, 0f3F800000;" : "+f"(a)); }
    if (V == 1) { a = ex2(a); }
    if (V == 2) { a = lg2(a); }
    if (V == 3) { a = __shfl_up_sync(0xffffffffu, a, 1); }
    if (V == 4) { unsigned r; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(u)); u = r; }
    if (V == 5) { a = lg2(1.f + ex2(-fabsf(a))); }
    if (V == 6) { asm volatile("max.f32 %0, %0, 0f3F800000;" : "+f"(a)); }
    if (V == 7) { a = __shfl_xor_sync(0xffffffffu, a, 1); }
  }
  long long t1 = clock64();
  io[threadIdx.x] = a + (float)u;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int V> void run(const char* name, float* io, long long* cyc) {
  const int n = 4096;
  long long h;
  for (int r = 0; r < 2; ++r) k<V><<<1, 32>>>(n, io, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-14s %6.1f cycles\n", name, (double)h / n);
}
int main() {
  float* io; long long* cyc;
  cudaMalloc(&io, 4096); cudaMemset(io, 0, 4096); cudaMalloc(&cyc, 8);
  run<0>("fadd", io, cyc); run<6>("fmnmx", io, cyc); run<1>("mufu.ex2", io, cyc); run<2>("mufu.lg2", io, cyc);
  run<3>("shfl.up", io, cyc); run<7>("shfl.bfly", io, cyc); run<4>("lds", io, cyc); run<5>("lse-core", io, cyc);
  return 0;
}
