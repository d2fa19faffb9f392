// tcgen05 bring-up probe (debug tool, not product): TMEM alloc / st / ld round
// trip, then one kind::tf32 MMA 128x128x8 from hand-built 128B-swizzled
// K-major and MN-major tiles, checked against a CPU product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tcgen05_probe tcgen05_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ uint64_t mkdesc(const void* p, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

// byte offset of element (r, c) (c = 0..31 fp32 within a 128-byte row) in a 128B-swizzled region of rows
__host__ __device__ unsigned swz(unsigned r, unsigned c) {
  const unsigned chunk = (c / 4) ^ (r % 8);
  return r * 128 + chunk * 16 + (c % 4) * 4;
}

__global__ void probe(const float* A, const float* B, float* D, unsigned* info, int mode, unsigned lbo, unsigned sbo) {
  // A: 128 (M) x 8 (K) row-major, B: 8 (K) x 128 (N) row-major. D: 128 x 128.
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* ta = (float*)smem;            // 16 KB
  float* tb = (float*)(smem + 16384);  // 16 KB
  uint64_t* bar = (uint64_t*)(smem + 32768);
  uint32_t* slot = (uint32_t*)(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 8192; i += blockDim.x) ((float*)smem)[i] = 0.f;
  __syncthreads();
  // K-major A: row m (128), k in 0..7 -> 128B row m, element k
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    int m = i / 8, k = i % 8;
    *(float*)((char*)ta + swz(m, k)) = A[m * 8 + k];
  }
  if (mode == 0) {  // B K-major: row n (128), element k
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
      int n = i / 8, k = i % 8;
      *(float*)((char*)tb + swz(n, k)) = B[k * 128 + n];
    }
  } else {  // B MN-major: chunk of 32 n at 4 KB; within: row k, element n%32
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
      int k = i / 128, n = i % 128;
      *(float*)((char*)tb + (n / 32) * 4096 + swz(k, n % 32)) = B[k * 128 + n];
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA reads)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  if (tid == 0) info[0] = tmem;
  if (warp == 0 && lane == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)mode << 16) | ((128u >> 3) << 17) |
                           ((128u >> 4) << 24);
    const uint64_t da = mkdesc(ta, 16, 1024);
    const uint64_t db = mode == 0 ? mkdesc(tb, 16, 1024) : mkdesc(tb, lbo, sbo);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
  }
  // wait
  {
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(su32(bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warps 0..3 read lanes 32w..32w+31
  if (warp < 4) {
    for (int c0 = 0; c0 < 128; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * 128 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(128 * 8), B(8 * 128), D(128 * 128);
  for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 7) % 13 - 6) / 8.f;
  for (int i = 0; i < 8 * 128; ++i) B[i] = (float)((i * 5) % 11 - 5) / 4.f;
  float *dA, *dB, *dD;
  unsigned* dI;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMalloc(&dI, 64);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const unsigned variants[][3] = {{0, 16, 1024}, {1, 4096, 1024}, {1, 1024, 4096}, {1, 4096, 128}, {1, 128, 4096}, {1, 16, 4096}, {1, 4096, 16}};
  for (auto& v : variants) {
    const int mode = v[0];
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 40000>>>(dA, dB, dD, dI, mode, v[1], v[2]);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned info[4];
    cudaMemcpy(info, dI, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    int nz = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double r = 0;
        for (int k = 0; k < 8; ++k) r += (double)A[m * 8 + k] * B[k * 128 + n];
        maxerr = fmax(maxerr, fabs(r - D[m * 128 + n]));
        maxref = fmax(maxref, fabs(r));
        nz += D[m * 128 + n] != 0.f;
      }
    printf("lbo %u sbo %u ", v[1], v[2]);
    printf("mode %d (%s B): err %s, tmem=%u, max err %.3e (max ref %.3e), nonzero %d, D[0..3] %g %g %g %g\n", mode,
           mode ? "MN-major" : "K-major", cudaGetErrorString(e), info[0], maxerr, maxref, nz, D[0], D[1], D[2], D[3]);
  }
  return 0;
}
