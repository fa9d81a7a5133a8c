// microbench.cu — engine peaks on the B200 that define the roofline denominators for the
// bit GEMMs (the "measured b1 peak" of the north star; NVIDIA publishes none), plus a
// layout probe that checks the tcgen05 operand layouts the kernels rely on.
//
//   b1_mma_sync : mma.sync.m16n8k256 .b1 xor.popc (ptxas emulates it on sm_100a with
//                 IMMA.16832 + MOVM — SURVEY §0.3)
//   s8_mma_sync : mma.sync.m16n8k32 s8 (legacy warp-level tensor path)
//   tc_i8_*     : tcgen05.mma kind::i8 M128, A from TMEM or SMEM (UTCIMMA)
//   popc        : LOP3 + POPC on 64-bit words (the CUDA-core engine)
//   dfma/dadd   : FP64 pipe (first layer)
// Prints one JSON object. Build: make -C paper_2006_16578_b200/csrc microbench.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "umma.cuh"

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

using namespace umma;

__host__ __device__ inline int probe_val(int m, int k) { return ((m * 7 + k * 3) % 61) + 1; }
__device__ inline uint32_t kmajor_off(int row, int k, int sbo) { return (row / 8) * sbo + (k / 16) * 128 + (row % 8) * 16 + k % 16; }

// D[m][n] = sum_k A[m][k] * B[n][k] with B one-hot (B[n][k] = n == k): D[m][n] = A[m][n].
__global__ void probe_kernel(int32_t* out_ts, int32_t* out_ss) {
  __shared__ __align__(1024) uint8_t bs[32 * 32];
  __shared__ __align__(1024) uint8_t as[128 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc(&tbase, 64);
  for (int i = tid; i < 32 * 32; i += 128) bs[kmajor_off(i / 32, i % 32, 256)] = (i / 32 == i % 32);
  for (int i = tid; i < 128 * 32; i += 128) as[kmajor_off(i / 32, i % 32, 256)] = (uint8_t)probe_val(i / 32, i % 32);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  uint32_t v[32];
  for (int c = 0; c < 8; ++c) {
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) w |= (uint32_t)probe_val(tid, 4 * c + b) << (8 * b);
    v[c] = w;
  }
  tmem_st8(taddr(tb, warp * 32, 32), v);
  tmem_st_wait();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t id = idesc_i8(128, 32);
  const uint64_t bd = sdesc(smem_u32(bs), 128, 256);
  if (tid == 0) {
    mma_i8_ts(tb, tb + 32, bd, id, 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  tmem_ld32(taddr(tb, warp * 32, 0), v);
  tmem_ld_wait();
  for (int n = 0; n < 32; ++n) out_ts[tid * 32 + n] = (int32_t)v[n];
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    mma_i8_ss(tb, sdesc(smem_u32(as), 128, 256), bd, id, 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 1);
  fence_after();
  tmem_ld32(taddr(tb, warp * 32, 0), v);
  tmem_ld_wait();
  for (int n = 0; n < 32; ++n) out_ss[tid * 32 + n] = (int32_t)v[n];
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 64);
}

// SS-mode with the halo kernel's SWIZZLE_64B layout: rows of 64 B, iters x 4 MMAs that
// alternate the two 32-byte K halves of the row.
template <int N>
__global__ void __launch_bounds__(128, 1) tc_sw64_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* as = smem;             // 128 x 64 bytes
  uint8_t* bs = smem + 128 * 64;  // N x 64 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  for (int i = tid; i < (128 + N) * 64 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N);
    const uint64_t ad = sdesc_sw(smem_u32(as), 64), bd = sdesc_sw(smem_u32(bs), 64);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_i8_ss(tb, ad + 2 * (j & 1), bd + 2 * (j & 1), id, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

// SS-mode with moving operands, as in a real GEMM: A walks 8 distinct 128x64-byte
// SWIZZLE_64B tiles (64 KB) and B 8 distinct Nx64-byte tiles, so no two consecutive MMAs read
// the same shared-memory bytes.
template <int N>
__global__ void __launch_bounds__(128, 1) tc_sw64_moving_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* as = smem;                 // 8 x 128 x 64 bytes
  uint8_t* bs = smem + 8 * 128 * 64;  // 8 x N x 64 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  for (int i = tid; i < 8 * (128 + N) * 64 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N);
    const uint64_t ad = sdesc_sw(smem_u32(as), 64), bd = sdesc_sw(smem_u32(bs), 64);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t k = (uint32_t)((it * 4 + j) & 15);  // tile (k>>1), K half (k&1)
        mma_i8_ss(tb, ad + (k >> 1) * (128 * 64 / 16) + 2 * (k & 1), bd + (k >> 1) * (N * 64 / 16) + 2 * (k & 1),
                  id, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

// The halo-mode MMA sequence of bgemm_tc_kernel (3x3 conv, C = 64, NI = 8 images x 16 sites):
// per unit 9 taps x 2 K halves, A = 128 rows at row offset (r*18 + s)*8 of a SWIZZLE_64B
// halo (multiples of 512 B), B = the tap's 64 x 64 block (4 KB apart), one accumulator.
// ALIGN1K pads the halo so every tap starts on a 1024-byte boundary (row offsets * 2).
template <int N, bool ALIGN1K, bool DENSE = false, bool TMEMLD = false, bool WARPWIDE = false, int COMMITS = 0,
          bool POLLERS = false>
__global__ void __launch_bounds__(576, 1) tc_halo_pattern_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* as = smem;               // halo: up to 2 * 56 * 512 bytes
  uint8_t* bs = smem + 56 * 1024;   // 9 x N x 64 bytes
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  for (int i = tid; i < (56 * 1024 + 9 * N * 64) / 16; i += 128) {
    if (DENSE) {  // random +-1 bytes (0x01 / 0xFF), like expanded activations and weights
      uint32_t w[4];
      for (int k = 0; k < 4; ++k) {
        uint32_t h = (uint32_t)(i * 4 + k) * 2654435761u;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        w[k] = 0x01010101u | ((h & 0x01010101u) * 0xFEu);
      }
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u, 0, 0, 0);
    }
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  if (WARPWIDE && warp == 0) {  // the kernel's issue style: whole warp loops, elect.sync issues
    const uint32_t id = idesc_i8(128, N);
    const uint64_t ad = sdesc_sw(smem_u32(as), 64), bd = sdesc_sw(smem_u32(bs), 64);
    uint32_t aoff[9];
    for (int t = 0; t < 9; ++t) aoff[t] = (uint32_t)(((t / 3) * 18 + t % 3) * 8 * 64 / 16);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        mma_i8_ss_w(tb, ad + aoff[t], bd + t * (N * 64 / 16), id, 1);
        mma_i8_ss_w(tb, ad + aoff[t] + 2, bd + t * (N * 64 / 16) + 2, id, 1);
      }
      // the kernel's per-unit commits (halo buffer free, accumulator full), never waited on here
      for (int c = 0; c < COMMITS; ++c) mma_commit_w(&bar2);
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
  } else if (!WARPWIDE && tid == 0) {
    const uint32_t id = idesc_i8(128, N);
    const uint64_t ad = sdesc_sw(smem_u32(as), 64), bd = sdesc_sw(smem_u32(bs), 64);
    uint32_t aoff[9];
    for (int t = 0; t < 9; ++t) aoff[t] = (uint32_t)(((t / 3) * 18 + t % 3) * 8 * 64 / 16) * (ALIGN1K ? 2 : 1);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        mma_i8_ss(tb, ad + aoff[t], bd + t * (N * 64 / 16), id, 1);
        mma_i8_ss(tb, ad + aoff[t] + 2, bd + t * (N * 64 / 16) + 2, id, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  } else if (POLLERS && warp >= 1) {  // the kernel's waiting roles: poll an mbarrier meanwhile
    mbar_wait(&bar, 0);
  } else if (TMEMLD && warp >= 1) {
    // concurrent epilogue-like TMEM reads of another accumulator region (warps 1-3 read
    // lane quarters 1-3; columns 256..)
    uint32_t acc[32], sink = 0;
    for (int it = 0; it < iters / 4; ++it) {
      tmem_ld32(tb + ((uint32_t)(warp * 32) << 16) + 256 + (it & 7) * 32, acc);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) sink += acc[j];
    }
    if (sink == 0x12345678u) cycles[0] = 0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

// tcgen05 i8 throughput: one thread issues iters x 4 MMAs (M128 x N x K32) back to back.
// The exact first layer's MMA stream (kernels_first_tc.cu, AlexNet 11x11/4 geometry): A from
// SWIZZLE_NONE digit planes with overlapping windows (LBO 16 B, SBO 128 B), per tile 11 kernel
// rows x 2 K-steps x 6 digits x (128 / N) channel groups, B weight blocks 64 units apart.
template <int N>
__global__ void __launch_bounds__(128, 1) tc_fconv_pattern_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kPlane = 17 * 1024, kRows = 11, kK = 2;
  uint8_t* bs = smem + 6 * kPlane;  // weights: kRows * kK * 4 blocks of 32 channels x 32 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  for (int i = tid; i < (6 * kPlane + kRows * kK * 4 * 1024) / 16; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u, 0x01020304u, 0, 0x7f7f7f7fu);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N);
    const uint64_t a0 = sdesc(smem_u32(smem), 16, 128), b0 = sdesc(smem_u32(bs), 128, 256);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int grp = 0; grp < 128 / N; ++grp)
        for (int r = 0; r < kRows; ++r)
          for (int kc = 0; kc < kK; ++kc) {
            const uint32_t rowoff = (uint32_t)((r & 3) * 4 + (r >> 2)) * 1024;
            const uint64_t bd = b0 + (uint64_t)(((r * kK + kc) * 4 + grp * (N / 32)) * 64);
            const uint64_t ad = a0 + (uint64_t)((rowoff + kc * 32) >> 4);
#pragma unroll
            for (int d = 0; d < 6; ++d)
              mma_i8_ss(tb + (grp & 1) * 192 * (N / 32 == 1) + d * N, ad + (uint64_t)(d * kPlane / 16), bd, id,
                        (r | kc) != 0);
          }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

template <bool ATMEM, int N>
__global__ void __launch_bounds__(128, 1) tc_peak_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* as = smem;              // 128 x 128 bytes
  uint8_t* bs = smem + 128 * 128;  // N x 128 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  for (int i = tid; i < (128 + N) * 128 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x01010101u, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_i8(128, N);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t bd = sdesc(smem_u32(bs + j * 256), 128, 1024);
        if (ATMEM)
          mma_i8_ts(tb, tb + 256 + j * 8, bd, id, 1);
        else
          mma_i8_ss(tb, sdesc(smem_u32(as + j * 256), 128, 1024), bd, id, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

__global__ void b1_peak_kernel(int iters, int* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u + 1, a2 = a0 * 5u + 7, a3 = a0 ^ 0x5a5a5a5au, b0 = a0 * 9u, b1 = ~a0;
  int d[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void s8_peak_kernel(int iters, int* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u + 1, a2 = a0 * 5u + 7, a3 = a0 ^ 0x5a5a5a5au, b0 = a0 * 9u, b1 = ~a0;
  int d[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 0x7fffffff) out[0] = s;
}

// 8 independent (xor, popc, add) chains on 64-bit words: 64 bit-MACs per chain step.
__global__ void popc_peak_kernel(int iters, int* out) {
  uint64_t x[8];
  int acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = (uint64_t)(threadIdx.x + i) * 0x9e3779b97f4a7c15ull;
    acc[i] = 0;
  }
  for (int it = 0; it < iters; ++it) {
    const uint64_t y = (uint64_t)it * 0x2545F4914F6CDD1Dull;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t z = x[i] ^ y;
      acc[i] += __popc((uint32_t)z) + __popc((uint32_t)(z >> 32));
    }
  }
  int s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void dfma_peak_kernel(int iters, double* out) {
  double acc[8];
  const double m = 1.0 + 1e-12 * threadIdx.x, a = 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], m, a);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == -1.0) out[0] = s;
}

__global__ void dadd_peak_kernel(int iters, const double* xs, double* out) {
  double acc[8];
  double x = xs[threadIdx.x & 31];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __dadd_rn(acc[i], (it & 1) ? x : -x);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == -1.0) out[0] = s;
}

template <class F>
static float time_ms(F launch, int reps = 3) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0, clk_khz = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f", sms, clk_khz / 1e3);

  // ---- layout probe
  int32_t *d_ts, *d_ss;
  CK(cudaMalloc(&d_ts, 128 * 32 * 4));
  CK(cudaMalloc(&d_ss, 128 * 32 * 4));
  probe_kernel<<<1, 128>>>(d_ts, d_ss);
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> ts(128 * 32), ss(128 * 32);
  CK(cudaMemcpy(ts.data(), d_ts, ts.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ss.data(), d_ss, ss.size() * 4, cudaMemcpyDeviceToHost));
  int bad_ts = 0, bad_ss = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      bad_ts += ts[m * 32 + n] != probe_val(m, n);
      bad_ss += ss[m * 32 + n] != probe_val(m, n);
    }
  printf(", \"probe_tmemA_mismatch\": %d, \"probe_smemA_mismatch\": %d, \"probe_row0_tmemA\": [", bad_ts, bad_ss);
  for (int n = 0; n < 32; ++n) printf("%s%d", n ? "," : "", ts[n]);
  printf("], \"probe_row0_smemA\": [");
  for (int n = 0; n < 32; ++n) printf("%s%d", n ? "," : "", ss[n]);
  printf("], \"probe_row0_expect\": [");
  for (int n = 0; n < 32; ++n) printf("%s%d", n ? "," : "", probe_val(0, n));
  printf("]");

  int* d_i;
  double* d_d;
  long long* d_cyc;
  CK(cudaMalloc(&d_i, 64));
  CK(cudaMalloc(&d_d, 256 * 8));
  CK(cudaMemset(d_d, 0, 256 * 8));
  CK(cudaMalloc(&d_cyc, 4096 * 8));

  // ---- tcgen05 i8
  auto tc = [&](auto kern, int N, bool atmem, const char* name) {
    const int iters = 4096;
    const size_t smem = (128 + N) * 128;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const float ms = time_ms([&] { kern<<<sms, 128, smem>>>(iters, d_cyc); });
    std::vector<long long> cyc(sms);
    cudaMemcpy(cyc.data(), d_cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto c : cyc) mean += c;
    mean /= sms;
    const double macs = (double)iters * 4 * 128 * N * 32 * sms;
    printf(", \"%s\": {\"tmacs\": %.1f, \"tops\": %.1f, \"mac_per_clk_sm\": %.0f, \"ms\": %.3f}", name,
           macs / ms / 1e9, 2 * macs / ms / 1e9, (double)iters * 4 * 128 * N * 32 / mean, ms);
    (void)atmem;
  };
  tc(tc_peak_kernel<true, 256>, 256, true, "tc_i8_tmemA_n256");
  tc(tc_peak_kernel<false, 256>, 256, false, "tc_i8_smemA_n256");
  tc(tc_peak_kernel<true, 128>, 128, true, "tc_i8_tmemA_n128");
  tc(tc_peak_kernel<true, 64>, 64, true, "tc_i8_tmemA_n64");
  tc(tc_peak_kernel<false, 128>, 128, false, "tc_i8_smemA_n128");
  tc(tc_peak_kernel<false, 64>, 64, false, "tc_i8_smemA_n64");
  tc(tc_sw64_kernel<64>, 64, false, "tc_i8_smemA_sw64_n64");
  tc(tc_sw64_kernel<128>, 128, false, "tc_i8_smemA_sw64_n128");
  {
    auto tcm = [&](auto kern, int N, const char* name) {
      const int iters = 4096;
      const size_t smem = 8 * (128 + N) * 64;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const float ms = time_ms([&] { kern<<<sms, 128, smem>>>(iters, d_cyc); });
      std::vector<long long> cyc(sms);
      cudaMemcpy(cyc.data(), d_cyc, sms * 8, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto c : cyc) mean += c;
      mean /= sms;
      const double macs = (double)iters * 4 * 128 * N * 32 * sms;
      printf(", \"%s\": {\"tmacs\": %.1f, \"mac_per_clk_sm\": %.0f, \"clk_per_mma\": %.1f, \"ms\": %.3f}", name,
             macs / ms / 1e9, (double)iters * 4 * 128 * N * 32 / mean, mean / (iters * 4.0), ms);
    };
    tcm(tc_sw64_moving_kernel<64>, 64, "tc_i8_smemA_sw64_moving_n64");
    tcm(tc_sw64_moving_kernel<128>, 128, "tc_i8_smemA_sw64_moving_n128");
    auto tch = [&](auto kern, int N, const char* name, size_t smem_total = 0, int threads = 128) {
      const int iters = 2048;
      const size_t smem = smem_total ? smem_total : 56 * 1024 + 9 * N * 64;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const float ms = time_ms([&] { kern<<<sms, threads, smem>>>(iters, d_cyc); });
      std::vector<long long> cyc(sms);
      cudaMemcpy(cyc.data(), d_cyc, sms * 8, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto c : cyc) mean += c;
      mean /= sms;
      const double macs = (double)iters * 18 * 128 * N * 32 * sms;
      printf(", \"%s\": {\"tmacs\": %.1f, \"clk_per_mma\": %.1f, \"ms\": %.3f}", name, macs / ms / 1e9,
             mean / (iters * 18.0), ms);
    };
    auto tcf = [&](auto kern, int N, const char* name) {
      const int iters = 64;
      const size_t smem = 6 * 17 * 1024 + 11 * 2 * 4 * 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const float ms = time_ms([&] { kern<<<sms, 128, smem>>>(iters, d_cyc); });
      std::vector<long long> cyc(sms);
      cudaMemcpy(cyc.data(), d_cyc, sms * 8, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto c : cyc) mean += c;
      mean /= sms;
      const double mmas = (double)iters * 11 * 2 * 6 * (128 / N);
      printf(", \"%s\": {\"clk_per_mma\": %.1f, \"clk_per_tile\": %.0f, \"ms\": %.3f}", name, mean / mmas,
             mean / iters, ms);
    };
    tcf(tc_fconv_pattern_kernel<32>, 32, "tc_i8_first_conv_pattern_n32");
    tcf(tc_fconv_pattern_kernel<64>, 64, "tc_i8_first_conv_pattern_n64");
    tch(tc_halo_pattern_kernel<64, false>, 64, "tc_i8_halo_pattern_n64");
    tch(tc_halo_pattern_kernel<64, true>, 64, "tc_i8_halo_pattern_n64_align1k");
    tch(tc_halo_pattern_kernel<128, false>, 128, "tc_i8_halo_pattern_n128");
    tch(tc_halo_pattern_kernel<64, false, true>, 64, "tc_i8_halo_pattern_n64_dense_pm1");
    tch(tc_halo_pattern_kernel<64, false, true, true>, 64, "tc_i8_halo_pattern_n64_with_tmem_ld");
    tch(tc_halo_pattern_kernel<64, false, true, false, true>, 64, "tc_i8_halo_pattern_n64_warpwide_elect");
    tch(tc_halo_pattern_kernel<64, false, true, false, true, 2>, 64, "tc_i8_halo_pattern_n64_2commits_per_unit");
    tch(tc_halo_pattern_kernel<64, false, true, false, true, 2, true>, 64, "tc_i8_halo_pattern_n64_17_polling_warps",
        0, 576);
    tch(tc_halo_pattern_kernel<64, false, true, false, true>, 64, "tc_i8_halo_pattern_n64_smem200k", 200 * 1024);
    tch(tc_halo_pattern_kernel<64, false, true, false, true>, 64, "tc_i8_halo_pattern_n64_smem225k", 225 * 1024);
    tch(tc_halo_pattern_kernel<128, false, true>, 128, "tc_i8_halo_pattern_n128_dense_pm1");
  }

  // ---- legacy warp MMA, popc, fp64: grid 148*8 blocks x 256 threads
  const int blocks = sms * 8, threads = 256, it = 2048;
  const double warps = (double)blocks * threads / 32;
  float ms = time_ms([&] { b1_peak_kernel<<<blocks, threads>>>(it, d_i); });
  printf(", \"b1_mma_sync\": {\"t_bitmacs\": %.1f, \"t_bitops\": %.1f}", warps * it * 4 * 16 * 8 * 256 / ms / 1e9,
         2 * warps * it * 4 * 16 * 8 * 256 / ms / 1e9);
  ms = time_ms([&] { s8_peak_kernel<<<blocks, threads>>>(it, d_i); });
  printf(", \"s8_mma_sync\": {\"tmacs\": %.1f}", warps * it * 4 * 16 * 8 * 32 / ms / 1e9);
  ms = time_ms([&] { popc_peak_kernel<<<blocks, threads>>>(it * 4, d_i); });
  const double pbits = (double)blocks * threads * it * 4 * 8 * 64;
  printf(", \"popc\": {\"t_bitmacs\": %.1f, \"t_bitops\": %.1f}", pbits / ms / 1e9, 2 * pbits / ms / 1e9);
  ms = time_ms([&] { dfma_peak_kernel<<<blocks, threads>>>(it * 4, d_d); });
  printf(", \"dfma\": {\"tflops\": %.2f}", 2.0 * blocks * threads * it * 4 * 8 / ms / 1e9);
  ms = time_ms([&] { dadd_peak_kernel<<<blocks, threads>>>(it * 4, d_d, d_d + 128); });
  printf(", \"dadd\": {\"t_per_s\": %.2f}", 1.0 * blocks * threads * it * 4 * 8 / ms / 1e9);
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
