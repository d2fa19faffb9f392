// tput.cu -- per-SMSP issue cost of the chain step's instruction classes on
// sm_100a (design evidence): 8 independent chains per thread, one warp per
// SMSP; cycles per warp-instruction.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(int n, float* io, long long* cyc) {
  float a[8];
  unsigned u[8];
  for (int i = 0; i < 8; ++i) { a[i] = io[threadIdx.x + i]; u[i] = __float_as_uint(a[i]); }
  const float b = io[200], c = io[201];
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (V == 0) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (V == 1) asm volatile("add.f32 %0, %0, 0f3F800000;" : "+f"(a[i]));
      if (V == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      if (V == 3) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (V == 4) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %1; selp.f32 %0, %0, %1, p;}" : "+f"(a[i]) : "f"(b));
      if (V == 5) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(u[i]) : "r"(7u));
      if (V == 6) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(__float_as_uint(b)));
      if (V == 7) asm volatile("mul.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
      if (V == 8) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (V == 9) { if (i & 1) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b)); else asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b)); }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + (float)u[i];
  io[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int V> void run(const char* name, float* io, long long* cyc) {
  const int n = 2048;
  long long h;
  for (int r = 0; r < 2; ++r) k<V><<<1, 128>>>(n, io, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %5.2f cycles/warp-instr\n", name, (double)h / (n * 8));
}
int main() {
  float* io; long long* cyc;
  cudaMalloc(&io, 8192); cudaMemset(io, 0, 8192); cudaMalloc(&cyc, 8);
  run<0>("fadd r,r", io, cyc); run<1>("fadd r,imm", io, cyc); run<2>("ffma r,r,r", io, cyc);
  run<3>("fmnmx", io, cyc); run<4>("fsetp+fsel", io, cyc); run<5>("imad", io, cyc); run<6>("iadd", io, cyc);
  run<7>("fmul r,r", io, cyc); run<8>("mufu.ex2", io, cyc); run<9>("fadd/fmnmx mix", io, cyc);
  return 0;
}
