// fc_backward.cu -- the CTC gradient's first consumer: the output fully
// connected layer's backward pass on tcgen05 tensor cores (sm_100a).
//
// Reference: FullyConnectedLayer::backward (proj/src/nn.cpp:874-899) for the
// network's output layer (network.cpp:135: no clipped ReLU, no batch norm),
// fed by train_epoch's dlogits (trainer.cpp:155-171):
//   db += sum_rows dpre          (nn.cpp:886-890)
//   dW += dpre^T x               (matmul_tn, nn.cpp:894)
//   dx  = dpre W                 (matmul, nn.cpp:895)
// with dpre = the CTC gradient rows [T][B][A] read as rows x A (padded frames
// are zero rows, so they add nothing), x the layer's cached input rows x H,
// W the A x H weight. Here the gradient never leaves the device: the batch's
// CTC call writes it, these kernels consume it on the same stream.
//
// Both products run on the 5th-generation tensor cores: one thread issues
// tcgen05.mma (kind::tf32, fp32 accumulators in TMEM) on 128 x 128 tiles
// whose operands TMA streams into 128B-swizzled shared memory through a
// 1-4 stage mbarrier pipeline; four epilogue warps read the accumulators back
// with tcgen05.ld and store them (dx) or add them (dW, split over the rows:
// the contraction dimension is the T*B rows). tcgen05 kind::tf32 reads
// K-major operands only, so the MN-major operands of dW (dpre^T and x) are
// transposed per stage in shared memory by the epilogue warps, and W for dx
// is transposed once into the workspace.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <utility>
#include <cstdint>
#include <cstdlib>

#include "ds2ctc_internal.h"

namespace ds2ctc {
namespace {

constexpr int kTileM = 128;
constexpr int kTileK = 32;   // fp32 elements per 128-byte swizzle row
constexpr int kStagesMax = 4;  // pipeline depth; 3 when MN-major operands also need raw buffers
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2-5 epilogue
constexpr int kTileBytes = kTileM * kTileK * 4;  // 16 KB: the A tile of a stage (B: BN / 128 of it)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
// Bounded wait: a pipeline bug must fail the launch (trap), never hang the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  unsigned long long t0 = 0;
  for (unsigned n = 0;; ++n) {
    unsigned done;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(m)), "r"(parity)
        : "memory");
    if (done) return;
    if ((n & 1023) == 1023) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 2000000000ull) __trap();  // 2 s
    }
  }
}

// 2-D TMA tile load (coordinates in elements, innermost first) completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor (sm_100 "version 1"), 128B swizzle:
// start address, leading / stride byte offsets (all >> 4), layout type 2.
__device__ __forceinline__ uint64_t smem_desc(const void* p, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_u32(p) >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;                 // version
  d |= 2ull << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::tf32: fp32 accumulate, tf32 A and B.
__host__ __device__ constexpr uint32_t instr_desc(int bn) {
  return (1u << 4)                              // D format F32
         | (2u << 7) | (2u << 10)               // A, B format TF32, both K-major
         | (static_cast<uint32_t>(bn >> 3) << 17) | (static_cast<uint32_t>(kTileM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(static_cast<uint32_t>(accumulate))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// One operand tile (128 rows of the MMA's M or N x 32 of K) into stage memory.
// K-major: one box {32 K, 128 rows} straight into the MMA layout. MN-major:
// four boxes {32 MN, 32 K}, 4 KB apart, into the raw buffer for the transposer.
template <bool kMN, int ROWS>
__device__ __forceinline__ void load_tile(float* dst, const CUtensorMap* map, int mn0, int k0, uint64_t* bar) {
  if (!kMN) {
    tma_load_2d(dst, map, k0, mn0, bar);
  } else {
#pragma unroll
    for (int i = 0; i < ROWS / 32; ++i) tma_load_2d(dst + i * 32 * kTileK, map, mn0 + 32 * i, k0, bar);
  }
}

// Byte offset of (row, col) in a 128B-swizzled region of 128-byte rows
// (col = fp32 index 0..31): 16-byte chunk index XOR (row mod 8).
__device__ __forceinline__ unsigned swz(unsigned row, unsigned col) {
  return row * 128 + ((((col >> 2) ^ row) & 7) << 4) + ((col & 3) << 2);
}

// MN-major raw tile ([mn chunk][k row][32 mn], swizzled) -> K-major MMA tile
// ([mn row][32 k], swizzled); 128 threads. tcgen05 kind::tf32 reads K-major
// operands only (an MN-major B computes nothing: tools/microbench/tcgen05_probe.cu),
// and dpre^T, x in dW are MN-major in memory, so each stage is transposed here.
// Reads: one swizzled 128-byte row per k across the lanes (conflict-free);
// writes: one 16-byte chunk per lane (4 wavefronts per 512 bytes, the minimum).
template <int ROWS>
__device__ __forceinline__ void transpose_tile(const float* raw, float* kmaj, int t) {
  const char* rb = reinterpret_cast<const char*>(raw);
  char* kb = reinterpret_cast<char*>(kmaj);
  const int mn_lo = t & 31;  // lane within the 32-wide chunk
  constexpr int kChunks = ROWS / 32;
#pragma unroll
  for (int it = 0; it < 2 * kChunks; ++it) {  // (ROWS x 8 quads) / 128 threads
    const int chunk = it % kChunks;                          // MN chunk (32 rows of the MMA tile)
    const int kq = (t >> 5) + 4 * (it / kChunks);            // k quad 0..7
    const int mn = chunk * 32 + mn_lo;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = *reinterpret_cast<const float*>(rb + chunk * 4096 + swz(4 * kq + e, mn_lo));
    *reinterpret_cast<float4*>(kb + swz(mn, 4 * kq)) = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// Descriptor of K-step j (8 tf32 = 32 bytes of K) of a K-major tile: rows
// 128 B apart, 8-row groups 1 KB apart; K advances inside the swizzled row.
__device__ __forceinline__ uint64_t tile_desc(const float* tile, int j) {
  return smem_desc(reinterpret_cast<const char*>(tile) + 32 * j, 16, 1024);
}

// Epilogue staging row pitch (floats): 16-byte aligned rows whose float4
// writes (a quarter-warp per row) and float4 reads (a quarter-warp per row)
// hit distinct banks.
constexpr int kOutPitch = 36;

struct GemmArgs {
  int M, N;          // extent of D (M x N)
  int k_blocks;      // 32-wide K blocks per split
  int k_total;       // K extent (for the split range)
  float* out;        // row-major output with leading dimension ldo: D, or D^T when transposed
  long long ldo;
  int accumulate;    // 1: out += D (atomic, split-K safe); 0: out = D
  int transposed;    // 1: out[n][m] = D[m][n]
};

// One K-major stage: the epilogue's staging rows alias the operand tiles
// (the epilogue starts after the last MMA has read them and no TMA load
// follows), so more CTAs share an SM (dx: 52 -> 34 KB, 4 -> 5 CTAs per SM).
template <bool kAMN, bool kBMN, int STAGES>
__host__ __device__ constexpr bool alias_out() { return !(kAMN || kBMN) && STAGES == 1; }

template <bool kAMN, bool kBMN, int BN, int STAGES>
__host__ __device__ constexpr int gemm_smem() {
  return alias_out<kAMN, kBMN, STAGES>()
             ? ((kTileBytes + BN * kTileK * 4) > 4 * 32 * kOutPitch * 4 ? (kTileBytes + BN * kTileK * 4)
                                                                          : 4 * 32 * kOutPitch * 4) + 256 + 1024
             : STAGES * ((kTileBytes + BN * kTileK * 4) * (1 + (kAMN || kBMN))) + 4 * 32 * kOutPitch * 4 + 256 + 1024;
}

// D[M x N] (+)= A[M x K] . B[K x N]; blockIdx = (n tile, m tile, K split).
// STAGES: pipeline depth (1 when K is a single block: several CTAs then share
// an SM, so one CTA's epilogue stores overlap another's loads).
template <bool kAMN, bool kBMN, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, STAGES == 1 ? 5 : STAGES == 2 ? 2 : 1)
    k_fc_gemm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, GemmArgs g) {
  constexpr bool kTrans = kAMN || kBMN;
  constexpr int kStages = STAGES;
  constexpr int kBBytes = BN * kTileK * 4;
  constexpr int kTmemCols = BN < 32 ? 32 : BN;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KB alignment for the 128B-swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* a_tiles = reinterpret_cast<float*>(smem);
  float* b_tiles = reinterpret_cast<float*>(smem + kStages * kTileBytes);
  unsigned char* p = smem + kStages * (kTileBytes + kBBytes);
  float* a_raw = reinterpret_cast<float*>(p);
  if (kAMN) p += kStages * kTileBytes;
  float* b_raw = reinterpret_cast<float*>(p);
  if (kBMN) p += kStages * kBBytes;
  constexpr bool kAlias = alias_out<kAMN, kBMN, STAGES>();
  if (kAlias && kTileBytes + kBBytes < 4 * 32 * kOutPitch * 4) p = smem + 4 * 32 * kOutPitch * 4;
  // [4 warps][32][kOutPitch]; over the operand tiles when kAlias
  float* stage_out = kAlias ? reinterpret_cast<float*>(smem) : reinterpret_cast<float*>(p);
  uint64_t* full = reinterpret_cast<uint64_t*>(kAlias ? p : p + 4 * 32 * kOutPitch * 4);
  uint64_t* ready = full + kStages;   // transposed (MN-major operands only)
  uint64_t* empty = ready + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * kTileM;
  const int kb_begin = blockIdx.z * g.k_blocks;
  const int kb_end = min(kb_begin + g.k_blocks, (g.k_total + kTileK - 1) / kTileK);
  const int nkb = max(kb_end - kb_begin, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(ready + s, 4);  // one arrival per transposer warp
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 128 lanes x 128 fp32 columns of accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(empty + s, ((i / kStages) - 1) & 1);
      mbar_expect_tx(full + s, kTileBytes + kBBytes);
      const int k0 = (kb_begin + i) * kTileK;
      load_tile<kAMN, kTileM>((kAMN ? a_raw : a_tiles) + s * kTileM * kTileK, &map_a, m0, k0, full + s);
      load_tile<kBMN, BN>((kBMN ? b_raw : b_tiles) + s * BN * kTileK, &map_b, n0, k0, full + s);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer: one thread, tcgen05.mma kind::tf32 into TMEM ----
    constexpr uint32_t idesc = instr_desc(BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      mbar_wait((kTrans ? ready : full) + s, (i / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float* at = a_tiles + s * kTileM * kTileK;
      const float* bt = b_tiles + s * BN * kTileK;
#pragma unroll
      for (int j = 0; j < kTileK / 8; ++j) mma_tf32(tmem, tile_desc(at, j), tile_desc(bt, j), idesc, i > 0 || j > 0);
      mma_commit(empty + s);  // the stage is free once these MMAs have read it
    }
    mma_commit(done);  // accumulator complete (also fires with nkb == 0)
  } else if (warp >= 2) {
    const int t = threadIdx.x - 64;  // 0..127
    if (kTrans) {
      // ---- transposer: MN-major raw tiles -> K-major MMA tiles ----
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        mbar_wait(full + s, (i / kStages) & 1);
        if (kAMN) transpose_tile<kTileM>(a_raw + s * kTileM * kTileK, a_tiles + s * kTileM * kTileK, t);
        if (kBMN) transpose_tile<BN>(b_raw + s * BN * kTileK, b_tiles + s * BN * kTileK, t);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> the MMA's async reads
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(ready + s)) : "memory");
      }
    }
    if (nkb > 0) {
      // ---- epilogue: TMEM -> registers -> (transpose in smem) -> coalesced rows ----
      const int q = warp & 3;  // TMEM lane quarter this warp may access
      mbar_wait(done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float* buf = stage_out + (warp - 2) * 32 * kOutPitch;
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // lane = row (q * 32 + lane) of the tile: write its 32 columns, read back by column
        if (g.transposed) {
          // out[n][m]: for each n, the lanes (consecutive m) are consecutive words
          const int row = m0 + q * 32 + lane;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = n0 + c0 + j;
            if (row < g.M && col < g.N) {
              float* o = g.out + static_cast<long long>(col) * g.ldo + row;
              if (g.accumulate) atomicAdd(o, __uint_as_float(v[j]));
              else *o = __uint_as_float(v[j]);
            }
          }
          continue;
        }
        // lane = row: its 32 columns into the staging rows as float4; then a
        // quarter-warp per row reads them back as float4, so each store
        // instruction writes four full 128-byte row segments
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(buf + lane * kOutPitch + j) =
              make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                          __uint_as_float(v[j + 3]));
        __syncwarp();
        const int c4 = (lane & 7) * 4;
        const int col = n0 + c0 + c4;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = it * 4 + (lane >> 3);
          const int row = m0 + q * 32 + r;
          const float4 val = *reinterpret_cast<const float4*>(buf + r * kOutPitch + c4);
          if (row < g.M) {
            float* o = g.out + static_cast<long long>(row) * g.ldo + col;
            if (col + 3 < g.N && !g.accumulate) {
              *reinterpret_cast<float4*>(o) = val;  // ldo % 4 == 0 and a 16-byte aligned base (validated)
            } else {
              const float e[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (col + u < g.N) {
                  if (g.accumulate) atomicAdd(o + u, e[u]);
                  else o[u] = e[u];
                }
            }
          }
        }
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

// Transposes the A x H weight into the K-major [H][pitch] operand of dx (zero pad).
__global__ void k_transpose_w(const float* __restrict__ w, int A, int H, float* __restrict__ wt, int pitch) {
  __shared__ float tile[32][33];
  const int a0 = blockIdx.y * 32, h0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int a = a0 + r, h = h0 + threadIdx.x;
    tile[r][threadIdx.x] = (a < A && h < H) ? w[static_cast<long long>(a) * H + h] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int h = h0 + r, a = a0 + threadIdx.x;
    if (h < H && a < pitch) wt[static_cast<long long>(h) * pitch + a] = tile[threadIdx.x][r];
  }
}

// db[a] += sum_rows g[row][a]: per block a chunk of rows, one thread per column.
__global__ void k_bias_grad(const float* __restrict__ g, long long ldg, int rows, int A, int rows_per_block,
                            float* __restrict__ db) {
  const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < A; a += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = r0; r < r1; ++r) s += g[static_cast<long long>(r) * ldg + a];
    atomicAdd(db + a, s);
  }
}

// Small alphabets (A <= 32): one pass over the gradient rows that both
// re-pitches them to the TMA-legal 32 floats (zero fill; dst may be null when
// A % 4 == 0) and sums db. 256 threads = 8 rows x 32 columns per iteration,
// per-thread column sums, then the 8 row groups folded in shared memory.
__global__ void __launch_bounds__(256) k_pad_bias(const float* __restrict__ src, int A, long long rows,
                                                  float* __restrict__ dst, int pitch, float* __restrict__ db) {
  __shared__ float part[8][33];
  const int c = threadIdx.x & 31, rg = threadIdx.x >> 5;
  float acc = 0.f;
  for (long long r = blockIdx.x * 8LL + rg; r < rows; r += gridDim.x * 8LL) {
    const float v = c < A ? src[r * A + c] : 0.f;
    acc += v;
    if (dst != nullptr && c < pitch) dst[r * pitch + c] = v;
  }
  part[rg][c] = acc;
  __syncthreads();
  if (rg == 0 && db != nullptr && c < A) {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += part[i][c];
    atomicAdd(db + c, s);
  }
}

// Pads rows of width A to the TMA-legal pitch (multiple of 4 floats), zero fill.
__global__ void k_pad_rows(const float* __restrict__ src, int A, float* __restrict__ dst, int pitch, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / pitch;
    const int c = static_cast<int>(i - r * pitch);
    dst[i] = c < A ? src[r * A + c] : 0.f;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Row-major fp32 matrix [outer][inner] (pitch in floats), box {32, box_outer}, 128B swizzle.
bool make_map(CUtensorMap* m, const float* base, long long inner, long long outer, long long pitch, int box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 4};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool kAMN, bool kBMN, int BN, int STAGES>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& g, int splits, cudaStream_t s) {
  static int configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  constexpr int smem = gemm_smem<kAMN, kBMN, BN, STAGES>();
  static_assert(smem <= 232448, "k_fc_gemm stage rings exceed the 227 KB shared-memory opt-in");
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_fc_gemm<kAMN, kBMN, BN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured[dev] = 1;
  }
  const dim3 grid((g.N + BN - 1) / BN, (g.M + kTileM - 1) / kTileM, splits);
  k_fc_gemm<kAMN, kBMN, BN, STAGES><<<grid, kThreads, smem, s>>>(ma, mb, g);
  return cudaGetLastError();
}

}  // namespace

namespace {
size_t pad_bytes(int rows, int A) {
  return (A % 4 == 0) ? 0 : (static_cast<size_t>(rows) * ((A + 3) / 4 * 4) * sizeof(float) + 255) / 256 * 256;
}
}  // namespace

// [padded gradient rows (A % 4 != 0)] [W^T, H x pitch]
size_t fc_backward_workspace(int rows, int A, int H) {
  return pad_bytes(rows, A) + static_cast<size_t>(H) * ((A + 3) / 4 * 4) * sizeof(float);
}

// rows x A gradient g (pitch A), rows x H input x, A x H weight w.
int fc_backward(const float* g, const float* x, const float* w, float* dw, float* db, float* dx, int rows, int A,
                int H, void* workspace, int sm_count, void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  if (rows == 0) return cudaSuccess;
  // TMA needs 16-byte row pitches: pad the gradient rows when A % 4 != 0
  // (English: 29 -> 32 floats, 6 % of a small buffer; Mandarin 6000 is aligned).
  // The workspace always holds W^T for dx after the padded rows.
  const float* gp = g;
  long long ldg = A;
  if (A <= 32) {  // fused re-pitch + bias sum (one pass over the gradient)
    const int pitch = (A + 3) / 4 * 4;
    float* dst = A % 4 != 0 ? static_cast<float*>(workspace) : nullptr;
    const long long blocks = std::min<long long>((rows + 7) / 8, 4LL * sm_count);
    k_pad_bias<<<static_cast<unsigned>(blocks), 256, 0, s>>>(g, A, rows, dst, pitch, db);
    if (dst) {
      gp = dst;
      ldg = pitch;
    }
  } else if (A % 4 != 0) {
    const int pitch = (A + 3) / 4 * 4;
    const long long n = static_cast<long long>(rows) * pitch;
    k_pad_rows<<<static_cast<unsigned>(std::min<long long>((n + 255) / 256, 4LL * sm_count * 8)), 256, 0, s>>>(
        g, A, static_cast<float*>(workspace), pitch, n);
    gp = static_cast<const float*>(workspace);
    ldg = pitch;
  }
  if (db && A > 32) {
    const int rpb = 256;
    k_bias_grad<<<dim3((A + 255) / 256, (rows + rpb - 1) / rpb), 256, 0, s>>>(gp, ldg, rows, A, rpb, db);
  }
  // dW[A x H] += g^T x, K = rows (split so the grid fills the SMs). Small
  // alphabets (A <= 32) run it as dW^T = x^T g: M = H, N = A = one 32-wide
  // tile (no padding of A to 128), written transposed. Otherwise M = A, N = H.
  // Both operands are MN-major in memory (transposed per stage in smem).
  if (dw) {
    CUtensorMap ma, mb;
    const int kb = (rows + kTileK - 1) / kTileK;
    // K split: whole waves of the one-CTA-per-SM grid (a partial last wave
    // costs a full one: 20 tiles x 30 splits = 600 CTAs was 4.05 waves),
    // 2-5 waves, the fullest last wave winning (English dW 131 -> 118 us)
    // Small alphabets: two-stage dW CTAs, two per SM, so one CTA's handoffs
    // (transpose, MMA, refill) overlap the other's loads: 118 -> 110 us per
    // English dW (DS2CTC_FC_DW_STAGES=4: one four-stage CTA per SM).
    static const int dw_stages = [] {
      const char* v = std::getenv("DS2CTC_FC_DW_STAGES");
      return v != nullptr && std::atoi(v) == 4 ? 4 : 2;
    }();
    const int slots = sm_count * (A <= 32 && dw_stages == 2 ? 2 : 1);  // resident dW CTAs per wave
    auto split_for = [&](int tiles) {
      int best_sp = 1;
      double best_eff = -1.0;
      for (int w = 2; w <= 5; ++w) {
        const int sp = std::max(1, std::min(kb, w * slots / tiles));
        const int kpb = (kb + sp - 1) / sp;
        const int n = (kb + kpb - 1) / kpb;  // splits actually launched
        const long long ctas = static_cast<long long>(n) * tiles;
        const double eff = static_cast<double>(ctas) / (((ctas + slots - 1) / slots) * slots);
        if (eff > best_eff + 1e-9) {
          best_eff = eff;
          best_sp = sp;
        }
      }
      const int kpb = (kb + best_sp - 1) / best_sp;
      return std::make_pair((kb + kpb - 1) / kpb, kpb);
    };
    int e;
    if (A <= 32) {
      if (!make_map(&ma, x, H, rows, H, kTileK) || !make_map(&mb, gp, A, rows, ldg, kTileK))
        return cudaErrorInvalidValue;
      const auto sp = split_for((H + kTileM - 1) / kTileM);
      GemmArgs ga{H, A, sp.second, rows, dw, H, 1, 1};
      e = dw_stages == 2 ? launch_gemm<true, true, 32, 2>(ma, mb, ga, sp.first, s)
                         : launch_gemm<true, true, 32, 4>(ma, mb, ga, sp.first, s);
    } else {
      if (!make_map(&ma, gp, A, rows, ldg, kTileK) || !make_map(&mb, x, H, rows, H, kTileK))
        return cudaErrorInvalidValue;
      const auto sp = split_for(((A + kTileM - 1) / kTileM) * ((H + 127) / 128));
      GemmArgs ga{A, H, sp.second, rows, dw, H, 1, 0};
      e = launch_gemm<true, true, 128, 3>(ma, mb, ga, sp.first, s);
    }
    if (e != cudaSuccess) return e;
  }
  // dx[rows x H] = g W: A operand g (K = A contiguous -> K-major), B operand
  // W^T (transposed once into the workspace: K-major); K = A.
  if (dx) {
    const int pitch = (A + 3) / 4 * 4;
    float* wt = reinterpret_cast<float*>(static_cast<unsigned char*>(workspace) + pad_bytes(rows, A));
    k_transpose_w<<<dim3((H + 31) / 32, (pitch + 31) / 32), dim3(32, 8), 0, s>>>(w, A, H, wt, pitch);
    CUtensorMap ma, mb;
    if (!make_map(&ma, gp, A, rows, ldg, kTileM) || !make_map(&mb, wt, A, H, pitch, 128))
      return cudaErrorInvalidValue;
    GemmArgs gx{rows, H, (A + kTileK - 1) / kTileK, A, dx, H, 0, 0};
    const int e = A <= kTileK ? launch_gemm<false, false, 128, 1>(ma, mb, gx, 1, s)
                              : launch_gemm<false, false, 128, 4>(ma, mb, gx, 1, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ds2ctc
