// bmm_tc.cu — kernel-level BMM on packed operands (bmm_pm1 / bmm_raw / bmm_pm1_bin,
// bmm.hpp:204-274) as one tcgen05 kernel per call: no pre-expanded operand in HBM, no
// second launch.
//
// One CTA (16 warps) per 128 x 64 output tile (M rows of A, N columns of B), the whole inner
// dimension at once (Kp = K rounded up to 128 bits, <= 1536):
//   * B's 64 packed columns (Kp/8 bytes each, contiguous in ColPacked) are expanded to +-1
//     int8 straight into shared memory in the UMMA K-major canonical layout (8-row x 16-byte
//     core matrices, LBO 128 B, SBO Kp*8 B); bits past K expand to 0, so pad bits of A
//     contribute nothing;
//   * A's 128 packed rows are expanded by the same PRMT sign replication into TMEM (one row
//     per TMEM lane, tcgen05.st), so A never touches shared memory;
//   * one thread issues the Kp/32 tcgen05.mma kind::i8 (A from TMEM, B from smem,
//     M128 x N64 x K32, s32 accumulate into 64 TMEM columns) and commits to an mbarrier;
//   * the epilogue reads the exact +-1 dot v = K - 2 popc(a ^ b) per (row, column) and
//     writes int32 v (bmm_pm1), (K - v) / 2 = popc (bmm_raw) or the thresholded bit
//     (lo <= v <= hi, bmm_pm1_bin) packed into RowPacked output words.
// Both operands use the same K permutation (pm1.cuh), so the dot products are exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <cstdint>

#include "api_internal.cuh"
#include "bnmath.cuh"
#include "kernels.cuh"
#include "pm1.cuh"
#include "umma.cuh"

namespace btnn_gpu {

namespace bmmtc {
constexpr int kThreads = 512;
constexpr int kBM = 128, kBN = 64;
constexpr int kMaxKp = 1536;  // A in TMEM: Kp/4 columns + 64 accumulator columns <= 512
}  // namespace bmmtc

struct BmmTcArgs {
  const uint64_t* a;  // RowPacked M x Kp bits
  const uint64_t* b;  // ColPacked N x Kp bits
  int M, N, K, Kp;
  int mode;                // EPI_I32 (raw or pm1) or EPI_BITS
  int raw;                 // EPI_I32: (K - v) / 2
  int32_t* out;            // M x N int32
  double* rout;            // EPI_F64: M x N f64 bn(v) (the last layer's logits)
  const double *bn_mean, *bn_s, *bn_rcp, *bn_gamma, *bn_beta;  // EPI_F64
  uint32_t* out_bits;      // RowPacked M x (cwo * 64) bits, as 32-bit words
  int cwo32;               // output words (32-bit) per row
  const long long* thr_lo;  // EPI_BITS: per column lo / hi (nullptr: v >= 0)
  const long long* thr_hi;
  int32_t* labels;      // EPI_F64, N <= 64 (whole-K kernel): each row's argmax written too
  const uint8_t* bpre;  // pipelined kernel, PRE: B expanded to {0,1} blocks (bmm_expand_b01_kernel)
};

// Staging slot of 16-byte chunk c of packed row r (cpr chunks per row): c ^ (r & 7) when that
// stays inside the row (every power-of-two cpr >= 8 and any cpr for the chunks it maps), else c.
// The map is a bijection on [0, cpr): x = c ^ (r & 7) < cpr is taken only when it is, and
// pairs (c, x) swap; chunks whose partner is out of range keep their slot.
__device__ __forceinline__ int stage_slot(int r, int c, int cpr) {
  const int x = c ^ (r & 7);
  return x < cpr ? x : c;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

bool bmm_tc_supported(int M, int N, int K) {
  const int kp = (K + 127) / 128 * 128;
  return M >= 1 && N >= 1 && K >= 1 && kp <= bmmtc::kMaxKp;
}

// Timing experiments (BTNN_TIMING builds): clock64 phase stamps of CTA 0, thread 0.
__device__ unsigned long long g_bmm_ts[16];
__device__ unsigned long long g_bmm_cta[2 * 1024];  // per CTA: globaltimer at start / end
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BMM_STAMP(k) \
  if (BTNN_TIMING && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) g_bmm_ts[k] = clock64();

__global__ void __launch_bounds__(bmmtc::kThreads, 1) bmm_tc_kernel(const __grid_constant__ BmmTcArgs p) {
  using namespace umma;
  BMM_STAMP(0)
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  if (BTNN_TIMING && threadIdx.x == 0 && cta < 1024) g_bmm_cta[2 * cta] = gtimer();
  extern __shared__ __align__(1024) uint8_t smem[];  // B: 64 rows x Kp bytes, canonical K-major
  __shared__ uint64_t mma_done;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int2 thr[bmmtc::kBN];  // EPI_BITS: per column (lo, width) of the range test
  __shared__ double bnp[5][bmmtc::kBN];  // EPI_F64: per column mean, s, rcp, gamma, beta
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, part = warp >> 2;  // TMEM lane quarter, and which quarter of the work
  const int m0 = blockIdx.y * bmmtc::kBM, n0 = blockIdx.x * bmmtc::kBN;
  const int Kp = p.Kp;
  const uint32_t sbo = (uint32_t)Kp * 8;
  // Stage the packed tiles in shared memory with coalesced 16-byte cp.async (consecutive lanes
  // on consecutive 16-byte chunks of a row / column; rows of A and columns of B are contiguous
  // in RowPacked / ColPacked), issued first so their latency covers the setup below. Chunk c of
  // row r lands at slot stage_slot(r, c), so the per-row reads (one row per lane) are
  // bank-conflict-free.
  const int cpr = Kp / 128;  // 16-byte chunks per packed row
  uint8_t* a_stage = smem + (size_t)bmmtc::kBN * Kp;          // 128 rows x Kp/8 bytes
  uint8_t* b_stage = a_stage + (size_t)bmmtc::kBM * (Kp / 8);  // 64 columns x Kp/8 bytes
  // Programmatic dependent launch: the next kernel of the stream may start its prologue now;
  // B (weights / the second operand) is staged before waiting for the previous kernel, A (the
  // previous layer's output) and every global write after.
  grid_dep_launch();
  {
    const uint8_t* ga = reinterpret_cast<const uint8_t*>(p.a);
    const uint8_t* gb = reinterpret_cast<const uint8_t*>(p.b);
    for (int g = tid; g < bmmtc::kBN * cpr; g += bmmtc::kThreads) {
      const int r = g / cpr, c = g - r * cpr, col = n0 + r;
      const bool ok = col < p.N;
      cp_async16(smem_u32(b_stage + (size_t)r * (Kp / 8) + (size_t)stage_slot(r, c, cpr) * 16),
                 gb + ((size_t)(ok ? col : 0) * cpr + c) * 16, ok ? 16 : 0);
    }
    grid_dep_wait();
    for (int g = tid; g < bmmtc::kBM * cpr; g += bmmtc::kThreads) {
      const int r = g / cpr, c = g - r * cpr, row = m0 + r;
      const bool ok = row < p.M;
      cp_async16(smem_u32(a_stage + (size_t)r * (Kp / 8) + (size_t)stage_slot(r, c, cpr) * 16),
                 ga + ((size_t)(ok ? row : 0) * cpr + c) * 16, ok ? 16 : 0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&mma_done, 1);
    fence_mbar_init();
  }
  if (p.mode == EPI_BITS && tid < bmmtc::kBN) {
    // (v - lo) <= width in 32 bits, bounds clamped to +-2^30 (|v| <= K < 2^30); an empty
    // range never fires; no thresholds: v >= 0
    int lo32 = 0;
    uint32_t w = 1u << 30;
    const int n = min(n0 + tid, p.N - 1);
    if (p.thr_lo) {
      const long long l = p.thr_lo[n], h = p.thr_hi[n];
      const long long lc = l < -(1ll << 30) ? -(1ll << 30) : l, hc = h > (1ll << 30) ? (1ll << 30) : h;
      lo32 = lc > hc ? (1 << 30) + 1 : (int)lc;
      w = lc > hc ? 0u : (uint32_t)(hc - lc);
    }
    thr[tid] = make_int2(lo32, (int)w);
  }
  if (p.mode == EPI_F64 && tid < bmmtc::kBN) {
    const int n = min(n0 + tid, p.N - 1);
    bnp[0][tid] = p.bn_mean[n];
    bnp[1][tid] = p.bn_s[n];
    bnp[2][tid] = p.bn_rcp ? p.bn_rcp[n] : 0.0;
    bnp[3][tid] = p.bn_gamma[n];
    bnp[4][tid] = p.bn_beta[n];
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  BMM_STAMP(1)
  // Warp 0 allocates TMEM while warps 1-15 expand B: it only arrives (bar.arrive) on the
  // staging barrier, whose other 15 warps wait (bar.sync) for every thread's copies.
  if (warp == 0) {
    asm volatile("bar.arrive 1, %0;" ::"n"(bmmtc::kThreads) : "memory");
    tmem_alloc(&tmem_base_sh, 512);
    BMM_STAMP(2)
  } else {
    asm volatile("bar.sync 1, %0;" ::"n"(bmmtc::kThreads) : "memory");
    // ---- B -> +-1 bytes (0 past K) in shared memory, canonical K-major ----
    // item = (column n, chunk c): lanes on consecutive columns (n & 7 spans one core-matrix
    // row group: the 16-byte stores of 8 lanes cover all 32 banks)
    for (int g = tid - 32; g < bmmtc::kBN * cpr; g += bmmtc::kThreads - 32) {
      const int n = g & 63, c = g >> 6;
      const uint4 bits = *reinterpret_cast<const uint4*>(b_stage + (size_t)n * (Kp / 8) + stage_slot(n, c, cpr) * 16);
      const uint32_t w4[4] = {bits.x, bits.y, bits.z, bits.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = 4 * c + u;       // 32-bit word of the column
        const int rem = p.K - 32 * i;  // valid bits of this word
        uint32_t o[8];
        if (n0 + n < p.N && rem > 0) {
          expand_word(w4[u], o);
          if (rem < 32) {
            // byte k of word s holds bit 8k + 7 - s: zero the bytes of bits >= rem
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              uint32_t keep = 0;
#pragma unroll
              for (int k = 0; k < 4; ++k) keep |= (8 * k + 7 - s < rem ? 0xFFu : 0u) << (8 * k);
              o[s] &= keep;
            }
          }
        } else {
#pragma unroll
          for (int s = 0; s < 8; ++s) o[s] = 0u;
        }
        // K index 32i + 4s + k: core-matrix column 2i (s < 4) and 2i + 1 (s >= 4)
        uint8_t* dst = smem + (size_t)(n >> 3) * sbo + (size_t)(2 * i) * 128 + (n & 7) * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(dst + 128) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
  }
  fence_before();
  __syncthreads();  // the TMEM base is visible
  fence_after();
  BMM_STAMP(3)
  const uint32_t tbase = tmem_base_sh;
  const uint32_t a_col0 = bmmtc::kBN;  // A after the 64 accumulator columns
  // ---- A -> +-1 bytes in TMEM, one row per lane; warp: lane quarter q, chunks c = part mod 4 ----
  {
    const int r = q * 32 + lane;
    const uint8_t* arow = a_stage + (size_t)r * (Kp / 8);
    for (int c = part; c < cpr; c += 4) {
      const uint4 bits = *reinterpret_cast<const uint4*>(arow + stage_slot(r, c, cpr) * 16);
      uint32_t v[32];
      expand_word(bits.x, v);
      expand_word(bits.y, v + 8);
      expand_word(bits.z, v + 16);
      expand_word(bits.w, v + 24);
      tmem_st32(taddr(tbase, q * 32, a_col0 + 32 * c), v);
    }
    tmem_st_wait();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B read by the tensor core
  fence_before();
  __syncthreads();
  fence_after();
  BMM_STAMP(4)
  if (tid == 0) {
    // one thread, descriptors advanced by their start-address field (16-byte units)
    const uint32_t idesc = idesc_i8(bmmtc::kBM, bmmtc::kBN);
    const uint64_t b0 = sdesc(smem_u32(smem), 128, sbo);
    for (int j = 0; j < Kp / 32; ++j) mma_i8_ts(tbase, tbase + a_col0 + 8 * j, b0 + (uint64_t)(16 * j), idesc, j > 0);
    mma_commit(&mma_done);
  }
  BMM_STAMP(5)
  mbar_wait(&mma_done, 0);
  fence_after();
  BMM_STAMP(6)
  // ---- epilogue: warp (q, part) reads lane quarter q, columns part * 16 .. + 15 ----
  {
    const int r = q * 32 + lane, row = m0 + r, c0 = part * 16;
    uint32_t acc[16];
    tmem_ld16(taddr(tbase, q * 32, c0), acc);
    tmem_ld_wait();
    const int ncol = min(16, p.N - (n0 + c0));
    if (p.mode == EPI_BITS) {
      if (row < p.M && ncol > 0) {
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int2 t = thr[c0 + j];
          word |= (uint32_t)((uint32_t)((int)acc[j] - t.x) <= (uint32_t)t.y) << j;
        }
        if (ncol < 16) word &= (1u << ncol) - 1u;
        reinterpret_cast<uint16_t*>(p.out_bits)[(size_t)row * p.cwo32 * 2 + (n0 + c0) / 16] = (uint16_t)word;
      }
    } else if (p.mode == EPI_F64) {
      // bn (bnmath.cuh: the reference's (v - mean) / s * gamma + beta, exactly) -> f64 rows
      // through shared memory (B's expanded tile is dead): rows of 64 doubles at a 528-byte
      // pitch, then each warp instruction writes one full 512-byte output row segment
      constexpr int kPitch = 66;  // doubles per staged row
      double* st = reinterpret_cast<double*>(smem);
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        double2 y;
        y.x = bn_apply((double)(int)acc[j], bnp[0][c0 + j], bnp[1][c0 + j], bnp[2][c0 + j], bnp[3][c0 + j],
                       bnp[4][c0 + j]);
        y.y = bn_apply((double)(int)acc[j + 1], bnp[0][c0 + j + 1], bnp[1][c0 + j + 1], bnp[2][c0 + j + 1],
                       bnp[3][c0 + j + 1], bnp[4][c0 + j + 1]);
        *reinterpret_cast<double2*>(st + r * kPitch + c0 + j) = y;
      }
      __syncthreads();
      const bool vec = (p.N & 1) == 0 && n0 + bmmtc::kBN <= p.N;
      for (int rr = warp; rr < bmmtc::kBM; rr += bmmtc::kThreads / 32) {
        const int orow = m0 + rr;
        if (orow >= p.M) break;
        const int cc = lane * 2;
        double* dst = p.rout + (size_t)orow * p.N + n0 + cc;
        const double2 v = *reinterpret_cast<const double2*>(st + rr * kPitch + cc);
        if (vec) {
          *reinterpret_cast<double2*>(dst) = v;
        } else {
          if (n0 + cc < p.N) dst[0] = v.x;
          if (n0 + cc + 1 < p.N) dst[1] = v.y;
        }
        if (p.labels) {
          // the row's first-index argmax, as argmax_kernel / the sequential scan
          // (inference.hpp:177-184): every column of the row is in this tile (N <= 64)
          double bv = -INFINITY;
          int bi = INT_MAX;
          if (cc < p.N) { bv = v.x; bi = cc; }
          if (cc + 1 < p.N && (bi == INT_MAX || v.y > bv)) { bv = v.y; bi = cc + 1; }
#pragma unroll
          for (int off = 16; off; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
          }
          if (lane == 0) p.labels[orow] = bi;
        }
      }
    } else {
      // through shared memory (B's expanded tile is dead once the MMAs completed): rows of 64
      // int32 at a 272-byte pitch (16-byte stores of consecutive rows hit different banks),
      // then each warp instruction writes two full 256-byte output row segments
      constexpr int kPitch = 68;  // int32 per staged row
      int32_t* st = reinterpret_cast<int32_t*>(smem);
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        int4 v;
        v.x = p.raw ? (p.K - (int)acc[j]) / 2 : (int)acc[j];
        v.y = p.raw ? (p.K - (int)acc[j + 1]) / 2 : (int)acc[j + 1];
        v.z = p.raw ? (p.K - (int)acc[j + 2]) / 2 : (int)acc[j + 2];
        v.w = p.raw ? (p.K - (int)acc[j + 3]) / 2 : (int)acc[j + 3];
        *reinterpret_cast<int4*>(st + r * kPitch + c0 + j) = v;
      }
      __syncthreads();
      const bool vec = (p.N & 3) == 0 && n0 + bmmtc::kBN <= p.N;
      for (int rr = warp * 2 + (lane >> 4); rr < bmmtc::kBM; rr += 2 * (bmmtc::kThreads / 32)) {
        const int orow = m0 + rr;
        if (orow >= p.M) break;
        const int cc = (lane & 15) * 4;
        int32_t* dst = p.out + (size_t)orow * p.N + n0 + cc;
        const int4 v = *reinterpret_cast<const int4*>(st + rr * kPitch + cc);
        if (vec) {
          *reinterpret_cast<int4*>(dst) = v;
        } else {
          const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (n0 + cc + k < p.N) dst[k] = vv[k];
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  BMM_STAMP(7)
  if (warp == 0) tmem_dealloc(tbase, 512);
  BMM_STAMP(8)
  if (BTNN_TIMING && threadIdx.x == 0 && cta < 1024) g_bmm_cta[2 * cta + 1] = gtimer();
}

// act: RowPacked M x K (stride ru(K, 128) bits), filt: ColPacked N x K; the Epi carries the
// output (EPI_I32 raw / pm1 into out_i32, EPI_BITS into out_bits with optional thresholds).
void launch_bmm_tc(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st) {
  BmmTcArgs p{};
  if (e.mode == EPI_F64 && e.labels && N <= bmmtc::kBN) {  // fused argmax
    p.labels = e.labels;
    if (e.labels_done) *e.labels_done = true;
  }
  p.a = a;
  p.b = b;
  p.M = M;
  p.N = N;
  p.K = K;
  p.Kp = (K + 127) / 128 * 128;
  p.mode = e.mode;
  p.raw = e.raw;
  p.out = e.out_i32;
  p.out_bits = reinterpret_cast<uint32_t*>(e.out_bits);
  p.cwo32 = (N + 127) / 128 * 4;
  p.thr_lo = e.thr_lo;
  p.thr_hi = e.thr_hi;
  p.rout = e.rout;
  p.bn_mean = e.bn_mean;
  p.bn_s = e.bn_s;
  p.bn_rcp = e.bn_rcp;
  p.bn_gamma = e.bn_gamma;
  p.bn_beta = e.bn_beta;
  // One CTA per SM: each allocates all 512 TMEM columns, so a second co-resident CTA would
  // block in tcgen05.alloc until the first exits — request enough smem that two never fit.
  const int smem = std::max(bmmtc::kBN * p.Kp + (bmmtc::kBM + bmmtc::kBN) * p.Kp / 8, 120 * 1024);
  static thread_local int configured = -1;
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  if (configured != dev) {
    BT_CUDA(cudaFuncSetAttribute(bmm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 std::max(bmmtc::kBN * bmmtc::kMaxKp + (bmmtc::kBM + bmmtc::kBN) * bmmtc::kMaxKp / 8,
                                          120 * 1024)));
    configured = dev;
  }
  const dim3 grid((unsigned)((N + bmmtc::kBN - 1) / bmmtc::kBN), (unsigned)((M + bmmtc::kBM - 1) / bmmtc::kBM));
  launch_pdl(bmm_tc_kernel, grid, dim3(bmmtc::kThreads), (size_t)smem, st, p);
  note_tc_launch(e.mode == EPI_BITS ? "bmm_packed/bin" : e.mode == EPI_F64 ? "bmm_packed/bn" : "bmm_packed/i32",
                 (int)(grid.x * grid.y), (int)(grid.x * grid.y));
}

// ---------------------------------------------------------------------------------------------
// K-pipelined variant for any inner dimension (bmm_pipe_kernel<BN>): one 128 x BN output tile
// per CTA (two CTAs per SM for BN <= 128, one for BN = 256), warp-specialized, per K-step of
// 128 bits:
//   * A warps (4 or 8; TMEM lane quarter = warp % 4): each thread stages its row's 16 bytes
//     (or half of them) with its own cp.async kPD steps ahead, expands them to +-1 bytes and
//     stores them into the step's TMEM ring slot (tcgen05.st), counting the row's set bits
//     below K (pa);
//   * B warps (4 or 8): each thread stages one column's 16 bytes (or half) the same way and
//     expands them to {0,1} bytes (bit set -> 1, bits past K -> 0: two instructions per output
//     word) into the step's shared-memory ring slot (canonical K-major, 8 core columns of 16 B
//     per 8-column group);
//   * one MMA warp waits for both halves of a slot, issues the four M128 x BN x K32 kind::i8
//     MMAs (A from TMEM) and commits them to the slot's empty barrier.
// No thread waits for another thread's staging: the only cross-warp handshakes are the ring's
// full / empty mbarriers. The accumulator holds d = sum(a * b01); the +-1 dot is
// v = sum(a) - 2 d = K - 2 pa - 2 d, read at the end by all producer warps with the epilogues of
// bmm_tc_kernel (int32 / thresholded bits / exact bn logits).
namespace bmmp {
constexpr int kR = 4;          // ring depth: expanded B slots (smem) and A slots (TMEM)
constexpr int kPD = 4;         // packed-bit prefetch distance in K-steps
constexpr int kPS = kPD + 1;   // packed staging slots per thread
template <int BN, bool PRE>
struct Cfg {
  // producer warps form kSG step groups (group g takes K-steps g, g + kSG, ...), so a warp's
  // serial per-step chain (stage -> expand -> store -> arrive) may take kSG MMA steps
  static constexpr int kSG = BN == 256 ? 2 : 1;
  static constexpr int kAW = 4 * kSG;                          // A warps (a row's 4 words each)
  // B warps per step group (PRE: none; one loader warp copies the pre-expanded blocks)
  static constexpr int kBWG = PRE ? 0 : BN / 32 > 4 ? BN / 32 : 4;
  static constexpr int kBW = kBWG * kSG;                       // B warps
  static constexpr int kPW = kAW + kBW + (PRE ? 1 : 0);        // producer warps
  static constexpr int kEW = PRE ? kAW : BN == 256 ? 16 : 8;   // epilogue warps (the first ones)
  static constexpr int kHG = kEW / 4;                          // epilogue warps per lane quarter
  static constexpr int kThreads = 32 * (kPW + 1);              // + the MMA warp
  static constexpr int kBWords = PRE ? 4 : 4 * BN / (32 * kBWG);  // B words per thread per K-step
  static constexpr int kTmemCols = BN == 256 ? 512 : 256;  // BN accumulator + kR x 32 A columns
  static constexpr int kBSlot = BN * 128;                  // expanded B of one K-step
  static constexpr int kOffStage = kR * kBSlot;            // per-thread packed staging
  static constexpr int kMain = kOffStage + kPS * 32 * (kAW + kBW) * 16;
  static constexpr int kEpi = 128 * 68 * 8;                // epilogue staging: 128 x 64 columns
  static constexpr int kMax = kMain > kEpi ? kMain : kEpi;
  // >= 80 KB: at most two CTAs per SM, so their TMEM allocations always fit
  static constexpr int kBytes = kMax > 80 * 1024 ? kMax : 80 * 1024;
};
}  // namespace bmmp

template <int BN, bool PRE>
__global__ void __launch_bounds__(bmmp::Cfg<BN, PRE>::kThreads, BN == 256 ? 1 : 2)
    bmm_pipe_kernel(const __grid_constant__ BmmTcArgs p) {
  using namespace umma;
  using L = bmmp::Cfg<BN, PRE>;
  constexpr int kThreads = L::kThreads, kHG = L::kHG, kR = bmmp::kR, kPD = bmmp::kPD, kPS = bmmp::kPS;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_a[kR], full_b[kR], empty[kR], acc_done;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int2 thr[BN];
  __shared__ double bnp[5][BN];
  __shared__ int pa_sh[L::kSG][128];  // per A row: set bits below K, per step group
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * 128, n0 = blockIdx.x * BN;
  const int KS = p.Kp / 128;  // K-steps = 16-byte chunks per packed row
  uint8_t* bring = smem;
  const uint8_t* ga = reinterpret_cast<const uint8_t*>(p.a);
  const uint8_t* gb = reinterpret_cast<const uint8_t*>(p.b);
  if (tid == 0) {
    for (int r = 0; r < kR; ++r) {
      mbar_init(&full_a[r], 4);
      mbar_init(&full_b[r], PRE ? 1 : L::kBWG);
      mbar_init(&empty[r], 1);
    }
    mbar_init(&acc_done, 1);
    fence_mbar_init();
  }
  if (p.mode == EPI_BITS && tid < BN) {  // (v - lo) <= width, as in bmm_tc_kernel
    int lo32 = 0;
    uint32_t w = 1u << 30;
    const int n = min(n0 + tid, p.N - 1);
    if (p.thr_lo) {
      const long long l = p.thr_lo[n], hh = p.thr_hi[n];
      const long long lc = l < -(1ll << 30) ? -(1ll << 30) : l, hc = hh > (1ll << 30) ? (1ll << 30) : hh;
      lo32 = lc > hc ? (1 << 30) + 1 : (int)lc;
      w = lc > hc ? 0u : (uint32_t)(hc - lc);
    }
    thr[tid] = make_int2(lo32, (int)w);
  }
  if (p.mode == EPI_F64 && tid < BN) {
    const int n = min(n0 + tid, p.N - 1);
    bnp[0][tid] = p.bn_mean[n];
    bnp[1][tid] = p.bn_s[n];
    bnp[2][tid] = p.bn_rcp ? p.bn_rcp[n] : 0.0;
    bnp[3][tid] = p.bn_gamma[n];
    bnp[4][tid] = p.bn_beta[n];
  }
  if (warp == 0) tmem_alloc(&tmem_base_sh, L::kTmemCols);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = tmem_base_sh;
  int pa = 0;
  auto valid = [](int r_) { return r_ >= 32 ? ~0u : r_ > 0 ? (1u << r_) - 1u : 0u; };
  constexpr int SG = L::kSG;
  if (warp < L::kAW) {
    // ================= A producers: row q*32 + lane, the K-steps of step group g =================
    const int q = warp & 3, g = warp >> 2, row = q * 32 + lane;
    const bool ok = m0 + row < p.M;
    const uint8_t* src = ga + (size_t)(ok ? m0 + row : 0) * KS * 16;
    uint8_t* stg = smem + L::kOffStage + (size_t)tid * kPS * 16;
    auto issue = [&](int i) {  // this thread's i-th K-step, s = g + i*SG
      const int s = g + i * SG;
      if (s < KS) cp_async16(smem_u32(stg + (i % kPS) * 16), src + (size_t)s * 16, ok ? 16 : 0);
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int i = 0; i < kPD; ++i) issue(i);
    for (int i = 0, s = g; s < KS; ++i, s += SG) {
      issue(i + kPD);
      asm volatile("cp.async.wait_group %0;" ::"n"(kPD) : "memory");
      const int r = s % kR;
      uint32_t v[32];
      const uint4 b4 = *reinterpret_cast<const uint4*>(stg + (i % kPS) * 16);
      const uint32_t w[4] = {b4.x, b4.y, b4.z, b4.w};
      const int rem = p.K - 128 * s;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        expand_word(w[k], v + 8 * k);
        pa += __popc(w[k] & valid(rem - 32 * k));
      }
      if (s >= kR) mbar_wait(&empty[r], (uint32_t)((s / kR - 1) & 1));  // MMAs of step s - kR done
      tmem_st32(taddr(tbase, q * 32, (uint32_t)(BN + r * 32)), v);
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[r]);
    }
    pa_sh[g][row] = pa;
  } else if (PRE && warp == L::kAW) {
    // ================= B loader: one bulk copy per K-step of the pre-expanded block =================
    if (lane == 0) {
      const uint8_t* src = p.bpre + (size_t)blockIdx.x * KS * L::kBSlot;
      for (int s = 0; s < KS; ++s) {
        const int r = s % kR;
        if (s >= kR) mbar_wait(&empty[r], (uint32_t)((s / kR - 1) & 1));
        mbar_arrive_expect_tx(&full_b[r], (uint32_t)L::kBSlot);
        constexpr int kChunk = L::kBSlot < 16384 ? L::kBSlot : 16384;
#pragma unroll
        for (int off = 0; off < L::kBSlot; off += kChunk)
          bulk_g2s(bring + (size_t)r * L::kBSlot + off, src + (size_t)s * L::kBSlot + off, (uint32_t)kChunk, &full_b[r]);
      }
    }
  } else if (!PRE && warp < L::kPW) {
    // ================= B producers: column n, words bg*kBWords .. of the K-steps of group g =================
    const int bt = tid - 32 * L::kAW;  // 0 .. 32*kBW - 1
    const int g = bt / (32 * L::kBWG), gt = bt % (32 * L::kBWG);
    constexpr int NWd = L::kBWords;
    const int n = gt % BN, bg = gt / BN;
    const bool ok = n0 + n < p.N;
    const uint8_t* src = gb + (size_t)(ok ? n0 + n : 0) * KS * 16 + bg * NWd * 4;
    uint8_t* stg = smem + L::kOffStage + (size_t)tid * kPS * 16;
    auto issue = [&](int i) {
      const int s = g + i * SG;
      if (s < KS) {
        if constexpr (NWd == 4) cp_async16(smem_u32(stg + (i % kPS) * 16), src + (size_t)s * 16, ok ? 16 : 0);
        else asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(stg + (i % kPS) * 16)),
                          "l"(src + (size_t)s * 16), "r"(ok ? 8 : 0) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int i = 0; i < kPD; ++i) issue(i);
    for (int i = 0, s = g; s < KS; ++i, s += SG) {
      issue(i + kPD);
      asm volatile("cp.async.wait_group %0;" ::"n"(kPD) : "memory");
      const int r = s % kR;
      uint32_t w[NWd];
      if constexpr (NWd == 4) {
        const uint4 b4 = *reinterpret_cast<const uint4*>(stg + (i % kPS) * 16);
        w[0] = b4.x; w[1] = b4.y; w[2] = b4.z; w[3] = b4.w;
      } else {
        const uint2 b2 = *reinterpret_cast<const uint2*>(stg + (i % kPS) * 16);
        w[0] = b2.x; w[1] = b2.y;
      }
      const int rem = p.K - 32 * (4 * s + bg * NWd);
      if (s >= kR) mbar_wait(&empty[r], (uint32_t)((s / kR - 1) & 1));
      uint8_t* dst = bring + (size_t)r * L::kBSlot + (n >> 3) * 1024 + (n & 7) * 16;
#pragma unroll
      for (int i = 0; i < NWd; ++i) {
        uint32_t o[8];
        expand_word01(w[i] & valid(rem - 32 * i), o);
        const int u = bg * NWd + i;  // word of the step: core columns 2u, 2u + 1
        *reinterpret_cast<uint4*>(dst + (2 * u) * 128) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(dst + (2 * u + 1) * 128) = make_uint4(o[4], o[5], o[6], o[7]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // read by the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_b[r]);
    }
  } else {
    // ================= MMA issuer =================
    const uint32_t idesc = idesc_i8(128, BN);
    for (int s = 0; s < KS; ++s) {
      const int r = s % kR;
      const uint32_t ph = (uint32_t)((s / kR) & 1);
      mbar_wait(&full_a[r], ph);
      mbar_wait(&full_b[r], ph);
      fence_after();
      const uint64_t b0 = sdesc(smem_u32(bring + (size_t)r * L::kBSlot), 128, 1024);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        mma_i8_ts_w(tbase, tbase + BN + r * 32 + 8 * j, b0 + (uint64_t)(16 * j), idesc, (s | j) != 0);
      mma_commit_w(&empty[r]);
    }
    mma_commit_w(&acc_done);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();  // pa_sh written
  mbar_wait(&acc_done, 0);
  fence_after();
  if (warp < L::kEW) {
    // ---- epilogue: warp (q, h) reads lane quarter q; v = kv - 2 d ----
    const int q = warp & 3, h = warp >> 2;
    const int rr0 = q * 32 + lane, row = m0 + rr0;
    int kv = p.K;
#pragma unroll
    for (int j = 0; j < SG; ++j) kv -= 2 * pa_sh[j][rr0];
    if (p.mode == EPI_BITS) {
#pragma unroll 1
      for (int c0 = h * (BN / kHG); c0 < (h + 1) * (BN / kHG); c0 += 16) {
        uint32_t acc[16];
        tmem_ld16(taddr(tbase, q * 32, c0), acc);
        tmem_ld_wait();
        const int ncol = min(16, p.N - (n0 + c0));
        if (row < p.M && ncol > 0) {
          uint32_t word = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int2 t = thr[c0 + j];
            word |= (uint32_t)((uint32_t)(kv - 2 * (int)acc[j] - t.x) <= (uint32_t)t.y) << j;
          }
          if (ncol < 16) word &= (1u << ncol) - 1u;
          reinterpret_cast<uint16_t*>(p.out_bits)[(size_t)row * p.cwo32 * 2 + (n0 + c0) / 16] = (uint16_t)word;
        }
      }
    }
  }
  if (p.mode != EPI_BITS) {
    // 64-column halves staged through shared memory (the rings are dead), then row-contiguous
    // stores by the producer warps: int32 rows at a 272-byte pitch, f64 rows at a 528-byte pitch
    constexpr int kEW = L::kEW, kCW = 64 / kHG;  // a warp's columns of the half
    const int q = warp & 3, h = warp >> 2;
    const int rr0 = q * 32 + lane;
    int kv = p.K;
    if (warp < kEW) {
#pragma unroll
      for (int j = 0; j < SG; ++j) kv -= 2 * pa_sh[j][rr0];
    }
#pragma unroll 1
    for (int hb = 0; hb < BN / 64; ++hb) {
      const int c0 = hb * 64 + h * kCW;
      if (warp < kEW) {
        uint32_t acc[kCW];
#pragma unroll
        for (int j = 0; j < kCW; j += 16) tmem_ld16(taddr(tbase, q * 32, c0 + j), acc + j);
        tmem_ld_wait();
        if (p.mode == EPI_F64) {
          double* st = reinterpret_cast<double*>(smem);
#pragma unroll
          for (int j = 0; j < kCW; j += 2) {
            double2 y;
            y.x = bn_apply((double)(kv - 2 * (int)acc[j]), bnp[0][c0 + j], bnp[1][c0 + j], bnp[2][c0 + j],
                           bnp[3][c0 + j], bnp[4][c0 + j]);
            y.y = bn_apply((double)(kv - 2 * (int)acc[j + 1]), bnp[0][c0 + j + 1], bnp[1][c0 + j + 1],
                           bnp[2][c0 + j + 1], bnp[3][c0 + j + 1], bnp[4][c0 + j + 1]);
            *reinterpret_cast<double2*>(st + rr0 * 66 + h * kCW + j) = y;
          }
        } else {
          int32_t* st = reinterpret_cast<int32_t*>(smem);
          // raw = popc(a ^ b) = (K - v) / 2
          const int m2 = p.raw ? 1 : -2, c2 = p.raw ? (p.K - kv) / 2 : kv;
#pragma unroll
          for (int j = 0; j < kCW; j += 4)
            *reinterpret_cast<int4*>(st + rr0 * 68 + h * kCW + j) =
                make_int4(c2 + m2 * (int)acc[j], c2 + m2 * (int)acc[j + 1], c2 + m2 * (int)acc[j + 2],
                          c2 + m2 * (int)acc[j + 3]);
        }
      }
      __syncthreads();
      const int nb = n0 + hb * 64;
      if (warp < kEW && p.mode == EPI_F64) {
        const double* st = reinterpret_cast<const double*>(smem);
        const bool vec = (p.N & 1) == 0 && nb + 64 <= p.N;
        for (int rr = warp; rr < 128; rr += kEW) {
          const int orow = m0 + rr;
          if (orow >= p.M) break;
          const int cc = lane * 2;
          double* dst = p.rout + (size_t)orow * p.N + nb + cc;
          const double2 v = *reinterpret_cast<const double2*>(st + rr * 66 + cc);
          if (vec) {
            *reinterpret_cast<double2*>(dst) = v;
          } else {
            if (nb + cc < p.N) dst[0] = v.x;
            if (nb + cc + 1 < p.N) dst[1] = v.y;
          }
        }
      } else if (warp < kEW) {
        const int32_t* st = reinterpret_cast<const int32_t*>(smem);
        const bool vec = (p.N & 3) == 0 && nb + 64 <= p.N;
        for (int rr = warp * 2 + (lane >> 4); rr < 128; rr += 2 * kEW) {
          const int orow = m0 + rr;
          if (orow >= p.M) break;
          const int cc = (lane & 15) * 4;
          int32_t* dst = p.out + (size_t)orow * p.N + nb + cc;
          const int4 v = *reinterpret_cast<const int4*>(st + rr * 68 + cc);
          if (vec) {
            *reinterpret_cast<int4*>(dst) = v;
          } else {
            const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (nb + cc + k < p.N) dst[k] = vv[k];
          }
        }
      }
      __syncthreads();  // the staging area is reused by the next half
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tbase, L::kTmemCols);
}

static BmmTcArgs bmm_args(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e) {
  BmmTcArgs p{};
  p.a = a;
  p.b = b;
  p.M = M;
  p.N = N;
  p.K = K;
  p.Kp = (K + 127) / 128 * 128;
  p.mode = e.mode;
  p.raw = e.raw;
  p.out = e.out_i32;
  p.out_bits = reinterpret_cast<uint32_t*>(e.out_bits);
  p.cwo32 = (N + 127) / 128 * 4;
  p.thr_lo = e.thr_lo;
  p.thr_hi = e.thr_hi;
  p.rout = e.rout;
  p.bn_mean = e.bn_mean;
  p.bn_s = e.bn_s;
  p.bn_rcp = e.bn_rcp;
  p.bn_gamma = e.bn_gamma;
  p.bn_beta = e.bn_beta;
  return p;
}

// B (ColPacked N x Kp bits) -> {0,1} byte blocks for the PRE kernel: block (N-tile t, K-step s)
// of BN columns x 128 bytes in the canonical K-major layout the MMA reads, bits past K and
// columns past N zero. One thread per (column, K-step): one 16-byte load, eight 16-byte stores
// (consecutive threads on consecutive columns: 128 contiguous bytes per 8 lanes).
__global__ void bmm_expand_b01_kernel(const uint4* __restrict__ b, int N, int K, int KS, int BN, int npad,
                                      uint8_t* __restrict__ out) {
  const long long item = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= (long long)npad * KS) return;
  const int n = (int)(item % npad), s = (int)(item / npad);
  const uint4 b4 = n < N ? __ldg(b + (size_t)n * KS + s) : make_uint4(0u, 0u, 0u, 0u);
  const uint32_t w4[4] = {b4.x, b4.y, b4.z, b4.w};
  const int t = n / BN, nn = n % BN;
  uint8_t* dst = out + ((size_t)t * KS + s) * BN * 128 + (nn >> 3) * 1024 + (nn & 7) * 16;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int rem = K - 32 * (4 * s + u);
    const uint32_t w = rem >= 32 ? w4[u] : rem > 0 ? w4[u] & ((1u << rem) - 1u) : 0u;
    uint32_t o[8];
    expand_word01(w, o);
    *reinterpret_cast<uint4*>(dst + (2 * u) * 128) = make_uint4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<uint4*>(dst + (2 * u + 1) * 128) = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

template <int BN, bool PRE>
static void launch_bmm_pipe_bn(const BmmTcArgs& p, cudaStream_t st) {
  using L = bmmp::Cfg<BN, PRE>;
  static thread_local int configured = -1;
  int dev = 0;
  BT_CUDA(cudaGetDevice(&dev));
  if (configured != dev) {
    BT_CUDA(cudaFuncSetAttribute(bmm_pipe_kernel<BN, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes));
    configured = dev;
  }
  const dim3 grid((unsigned)((p.N + BN - 1) / BN), (unsigned)((p.M + 127) / 128));
  bmm_pipe_kernel<BN, PRE><<<grid, L::kThreads, L::kBytes, st>>>(p);
  BT_CUDA(cudaGetLastError());
  note_tc_launch(p.mode == EPI_BITS ? "bmm_pipe/bin" : p.mode == EPI_F64 ? "bmm_pipe/bn" : "bmm_pipe/i32",
                 (int)(grid.x * grid.y), (int)(grid.x * grid.y));
}

// per host thread and device: the pre-expanded B workspace of the last call
struct BpreWs {
  int dev = -1;
  DevBuf buf;
};
static thread_local BpreWs g_bpre;

// Any M, N, K. 128 x 256 tiles (one CTA per SM, N = 256 MMAs) when they occupy at least half
// the SMs: with pre_b (kernel-level calls, which own the workspace for the duration of the call)
// B is expanded once into {0,1} blocks by bmm_expand_b01_kernel and streamed by bulk copies,
// else expanded in the GEMM by its own producer warps. Otherwise 128 x 128 tiles when they fill
// the two CTA slots per SM, else 128 x 64.
void launch_bmm_pipe(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st,
                     bool pre_b) {
  BmmTcArgs p = bmm_args(M, N, K, a, b, e);
  int dev = 0, sms = 148;
  BT_CUDA(cudaGetDevice(&dev));
  BT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long mt = (M + 127) / 128;
  if (2 * mt * ((N + 255) / 256) >= sms) {
    if (!pre_b) {
      launch_bmm_pipe_bn<256, false>(p, st);
      return;
    }
    const int KS = p.Kp / 128, npad = (N + 255) / 256 * 256;
    const size_t bytes = (size_t)npad * KS * 128;
    if (g_bpre.dev != dev || g_bpre.buf.bytes() < bytes) {
      g_bpre.buf.alloc(bytes);
      g_bpre.dev = dev;
    }
    const long long items = (long long)npad * KS;
    bmm_expand_b01_kernel<<<(unsigned)((items + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(b), N, K, KS, 256, npad, g_bpre.buf.get<uint8_t>());
    BT_CUDA(cudaGetLastError());
    p.bpre = g_bpre.buf.get<uint8_t>();
    launch_bmm_pipe_bn<256, true>(p, st);
  } else if (mt * ((N + 127) / 128) >= 2LL * sms) {
    launch_bmm_pipe_bn<128, false>(p, st);
  } else {
    launch_bmm_pipe_bn<64, false>(p, st);
  }
}

static std::atomic<int> g_bmm_kernel{BTNN_BMM_AUTO};

// Packed-operand BMM: the whole-K kernel when K fits it, else the K-pipelined one
// (btnn_cuda_set_bmm_kernel forces either).
const char* launch_bmm_packed(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e,
                              cudaStream_t st) {
  const int k = g_bmm_kernel.load();
  const bool whole = k == BTNN_BMM_WHOLE_K || (k == BTNN_BMM_AUTO && bmm_tc_supported(M, N, K));
  if (whole) {
    require(bmm_tc_supported(M, N, K), BTNN_UNSUPPORTED_SHAPE, "whole-K BMM kernel: K > 1536");
    launch_bmm_tc(M, N, K, a, b, e, st);
    return "tc_i8_bmm";
  }
  launch_bmm_pipe(M, N, K, a, b, e, st, k != BTNN_BMM_PIPELINED_NO_PRE);
  return "tc_i8_bmm_pipe";
}

// Fully-connected plan layers: the packed kernels when K fits the whole-K one, or when the
// pipelined one has at least one 128 x 64 tile per SM; nullptr leaves the layer to the
// split-K implicit GEMM (few output tiles, long K).
const char* launch_bmm_fc(int M, int N, int K, const uint64_t* a, const uint64_t* b, const Epi& e, cudaStream_t st) {
  const int k = g_bmm_kernel.load();
  if (k < BTNN_BMM_PIPELINED && bmm_tc_supported(M, N, K)) {
    launch_bmm_tc(M, N, K, a, b, e, st);
    return "tc_i8_bmm";
  }
  int dev = 0, sms = 148;
  BT_CUDA(cudaGetDevice(&dev));
  BT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long tiles = (long long)((M + 127) / 128) * ((N + 63) / 64);
  if (k >= BTNN_BMM_PIPELINED || (k == BTNN_BMM_AUTO && tiles >= sms)) {
    launch_bmm_pipe(M, N, K, a, b, e, st, false);  // (captured into plan graphs: no shared workspace)
    return "tc_i8_bmm_pipe";
  }
  return nullptr;
}

}  // namespace btnn_gpu

extern "C" int btnn_cuda_set_bmm_kernel(int which) {
  return btnn_gpu::guard([&] {
    btnn_gpu::require(which >= BTNN_BMM_AUTO && which <= BTNN_BMM_PIPELINED_NO_PRE, BTNN_INVALID_INPUT,
                      "set_bmm_kernel: unknown kernel");
    btnn_gpu::g_bmm_kernel.store(which);
  });
}

extern "C" int btnn_cuda_debug_bmm_timestamps(unsigned long long* out, size_t n) {
  return btnn_gpu::guard([&] {
    BT_CUDA(cudaDeviceSynchronize());
    BT_CUDA(cudaMemcpyFromSymbol(out, btnn_gpu::g_bmm_ts, (n < 16 ? n : 16) * 8));
    if (n >= 16 + 2048) BT_CUDA(cudaMemcpyFromSymbol(out + 16, btnn_gpu::g_bmm_cta, 2048 * 8));
  });
}
