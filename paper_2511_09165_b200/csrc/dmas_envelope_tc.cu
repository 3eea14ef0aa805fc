// K4 on the tensor cores — envelope low-pass as a banded Toeplitz contraction (tcgen05 + TMEM).
//
//   e[t] = max(0, sum_{j<L} h[j] |y[t + c - j]|),  c = (L-1)/2, zeros outside [0, T)
//   ("absolute value ... then low-pass filtered"; 5 kHz)
//
// View a row in blocks of 32 samples: t = 32 tau + n, s = 32 (tau + q) + k.  Then
//   E[tau][n] = sum_{q=-2}^{2} sum_{k<32} A[tau + q][k] * H_q[k][n],
//   A[tau][k] = |y[32 tau + k]|,  H_q[k][n] = h[n + c - 32 q - k]  (0 outside [0, L))
// i.e. five M=128 x N=32 x K=32 GEMMs per 4096-sample tile, where the block shift q is a 16-byte
// move of the A descriptor's start address (K-major, no swizzle, SBO = 16 B * 8 rows so every
// row is 16 B after the previous one).  MACs per output = 5 * 32 = 160 (127 useful).
//
// Precision: 3-pass split a = a_hi + a_lo, h = h_hi + h_lo; hi*hi + hi*lo + lo*hi with fp32
// accumulation in TMEM.  BF16 parts (kind::f16, K = 16 per MMA; default): relative error per
// product <= 2^-18 + 2^-17 ~ 1.1e-5, and since the taps are (all but 34 tiny ones) positive the
// summed error is <= ~1.1e-5 of the envelope value itself — 9x inside the 1e-4 bar.  TF32 parts
// (kind::tf32, K = 8): ~2^-21, at twice the MMA count.  Measured on B200: every tcgen05.mma with
// N <= 64 costs >= 44 cycles, so the MMA count (not the MAC count) is what the split type buys.
//
// Per CTA (persistent, 1 CTA / SM, warp-specialised, mbarrier pipelines): a TMA-producer warp
// keeps a 5-slot ring of raw row tiles filling (cp.async.bulk, complete_tx); 8 converter warps
// turn a tile into |.| hi/lo TF32 in the UMMA canonical layout (double-buffered A) and drain the
// previous tile's TMEM accumulator (tcgen05.ld -> clamp -> store); one MMA-issuer lane issues the
// tile's 60 tcgen05.mma into one of two TMEM accumulators and commits to an mbarrier — so TMA,
// tensor core and SIMT work overlap.

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "dmas_kernels.cuh"

namespace dmas {
namespace tc {

constexpr int BLK = 32;                 // samples per block (MMA N; K per shift)
constexpr int TILE_BLOCKS = 128;        // MMA M: blocks per tile
constexpr int TILE_T = BLK * TILE_BLOCKS;   // 4096 outputs per tile
constexpr int HALO = 2;                 // block shifts q in [-2, 2]
constexpr int NQ = 2 * HALO + 1;
constexpr int B_LBO = BLK * 16;         // 512
constexpr int STAGE_FLOATS = (TILE_BLOCKS + 2 * HALO) * BLK;   // 4224 raw samples per tile
constexpr int STAGE_BYTES = STAGE_FLOATS * 4;
constexpr int NSTAGE = 5;
constexpr int THREADS = 512;            // converter / epilogue threads (16 warps)
constexpr int TMEM_COLS = 64;           // two 32-column fp32 accumulators

// Operand element: BF16 (2 B, 8 per 16-byte core row, K = 16 per MMA) or TF32 (4 B, 4 per row, K = 8).
template <bool BF16> struct El {
  // A slots (>= TILE_BLOCKS + 2 HALO) padded so the converter's stores are bank-conflict free:
  // BF16 8-byte stores need LBO/4 = 8 mod 32 (138 slots), TF32 16-byte stores need 4 mod 32 (137).
  static constexpr int SLOTS = BF16 ? 138 : 137;
  static constexpr int A_LBO = SLOTS * 16;                      // bytes between K core columns of A
  static constexpr int BYTES = BF16 ? 2 : 4;
  static constexpr int PER_ROW = 16 / BYTES;                    // elements per 16-byte core row
  static constexpr int CORE_COLS = BLK / PER_ROW;               // core columns per block of K = 32
  static constexpr int K_MMA = BF16 ? 16 : 8;
  static constexpr int KSTEPS = BLK / K_MMA;
  static constexpr int A_BYTES = A_LBO * CORE_COLS;             // one split of one A buffer
  static constexpr int B_BYTES = B_LBO * CORE_COLS;             // one H_q split
  static constexpr int OFF_A = 0;                               // [2 buf][2 split][A_BYTES]
  static constexpr int OFF_B = OFF_A + 4 * A_BYTES;             // [2 split][NQ][B_BYTES]
  static constexpr int OFF_S = (OFF_B + 2 * NQ * B_BYTES + 1023) / 1024 * 1024;   // [NSTAGE][STAGE_BYTES]
  static constexpr int SMEM_BYTES = OFF_S + NSTAGE * STAGE_BYTES;
  // instruction descriptor: D f32, A/B bf16 (kind::f16) or tf32, K-major, N = 32, M = 128
  static constexpr uint32_t IDESC = (1u << 4) | ((BF16 ? 1u : 2u) << 7) | ((BF16 ? 1u : 2u) << 10) |
                                    ((uint32_t)(BLK >> 3) << 17) | ((128u >> 4) << 24);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
template <bool BF16>
__device__ __forceinline__ void mma_issue(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  if (BF16)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(El<true>::IDESC), "r"(accumulate));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(El<false>::IDESC), "r"(accumulate));
}
// hi / lo split of a non-negative-or-any float into two operand elements (raw bits)
template <bool BF16> __device__ __forceinline__ void split(float a, uint32_t& hi, uint32_t& lo);
template <> __device__ __forceinline__ void split<false>(float a, uint32_t& hi, uint32_t& lo) {
  hi = to_tf32(a);
  lo = to_tf32(a - __uint_as_float(hi));
}
template <> __device__ __forceinline__ void split<true>(float a, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 h = __float2bfloat16_rn(a);
  const __nv_bfloat16 l = __float2bfloat16_rn(a - __bfloat162float(h));
  hi = (uint32_t)__bfloat16_as_ushort(h);
  lo = (uint32_t)__bfloat16_as_ushort(l);
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

struct Tile {
  int64_t row, ts;   // row index, first output sample of the tile
};
__device__ __forceinline__ Tile tile_of(int64_t j, int64_t tiles_per_row) {
  Tile t;
  t.row = j / tiles_per_row;
  t.ts = (j - t.row * tiles_per_row) * TILE_T;
  return t;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp roles: warps 0..7 convert (stage -> |.| TF32 hi/lo A) and drain accumulators (epilogue);
// warp 8 lane 0 issues the tcgen05.mma; warp 9 lane 0 issues the TMA bulk loads.
template <bool BF16>
__global__ void __launch_bounds__(THREADS + 64, 1) k_envelope_tc(const float* __restrict__ y, float* __restrict__ out,
                                                                int64_t rows, int64_t T,
                                                                const __grid_constant__ LpTaps127 taps, int32_t L) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t stage_full[NSTAGE], stage_empty[NSTAGE];
  __shared__ __align__(8) uint64_t a_full[2], mma_done[2], d_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tiles_per_row = (T + TILE_T - 1) / TILE_T;
  const int64_t n_tiles = rows * tiles_per_row;
  const int64_t first = blockIdx.x, step = gridDim.x;
  const int64_t my_tiles = first < n_tiles ? (n_tiles - 1 - first) / step + 1 : 0;
  using E = El<BF16>;
  float* stage = reinterpret_cast<float*>(smem + E::OFF_S);

  // ---- one-time setup: barriers, TMEM, the constant Toeplitz blocks H_q (hi / lo TF32)
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&stage_full[s], 1);
      mbar_init(&stage_empty[s], THREADS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], THREADS);
      mbar_init(&mma_done[b], 1);
      mbar_init(&d_empty[b], THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int c = (L - 1) / 2;
  for (int e = tid; e < NQ * BLK * BLK; e += blockDim.x) {
    const int qi = e / (BLK * BLK), r = e - qi * BLK * BLK, n = r / BLK, k = r - n * BLK;
    const int q = qi - HALO;
    const int j = n + c - BLK * q - k;
    const float h = (j >= 0 && j < L) ? taps.h[j] : 0.f;
    uint32_t hi, lo;
    split<BF16>(h, hi, lo);
    const uint32_t off = (uint32_t)(qi * E::B_BYTES + n * 16 + (k / E::PER_ROW) * B_LBO + (k % E::PER_ROW) * E::BYTES);
    if (BF16) {
      *reinterpret_cast<uint16_t*>(smem + E::OFF_B + off) = (uint16_t)hi;
      *reinterpret_cast<uint16_t*>(smem + E::OFF_B + NQ * E::B_BYTES + off) = (uint16_t)lo;
    } else {
      *reinterpret_cast<uint32_t*>(smem + E::OFF_B + off) = hi;
      *reinterpret_cast<uint32_t*>(smem + E::OFF_B + NQ * E::B_BYTES + off) = lo;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == THREADS / 32 + 1) {
    // ================= TMA producer: raw samples [ts - 64, ts + 4160) of each tile
    if (lane == 0) {
      for (int64_t jj = 0; jj < my_tiles; ++jj) {
        const int slot = (int)(jj % NSTAGE);
        if (jj >= NSTAGE) mbar_wait(&stage_empty[slot], (uint32_t)(((jj - NSTAGE) / NSTAGE) & 1));
        const Tile tt = tile_of(first + jj * step, tiles_per_row);
        const int64_t lo_t = max((int64_t)0, tt.ts - HALO * BLK);
        const int64_t hi_t = min(T, tt.ts + TILE_T + HALO * BLK);
        const uint32_t bytes = (uint32_t)((hi_t - lo_t) * 4);
        mbar_expect_tx(&stage_full[slot], bytes);
        bulk_g2s(stage + slot * STAGE_FLOATS + (lo_t - (tt.ts - HALO * BLK)), y + tt.row * T + lo_t, bytes,
                 &stage_full[slot]);
      }
    }
  } else if (warp == THREADS / 32) {
    // ================= MMA issuer: 5 shifts x 4 K-steps x 3 split products per tile
    if (lane == 0) {
      const uint64_t a0 = smem_desc(smem_u32(smem + E::OFF_A), E::A_LBO, 128);
      const uint64_t b0 = smem_desc(smem_u32(smem + E::OFF_B), B_LBO, 128);
      for (int64_t jj = 0; jj < my_tiles; ++jj) {
        const int buf = (int)(jj & 1);
        mbar_wait(&a_full[buf], (uint32_t)((jj >> 1) & 1));
        if (jj >= 2) mbar_wait(&d_empty[buf], (uint32_t)(((jj - 2) >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem_base + (uint32_t)(buf * BLK);
        const uint64_t ab = a0 + (uint64_t)((2 * buf * E::A_BYTES) >> 4);
        uint32_t acc = 0;
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {           // lo*hi, hi*lo, hi*hi
          const uint64_t a_split = (pass == 0) ? (uint64_t)(E::A_BYTES >> 4) : 0;
          const uint64_t b_split = (pass == 1) ? (uint64_t)((NQ * E::B_BYTES) >> 4) : 0;
#pragma unroll
          for (int qi = 0; qi < NQ; ++qi) {
#pragma unroll
            for (int s = 0; s < E::KSTEPS; ++s) {        // K_MMA = 2 core columns
              mma_issue<BF16>(d, ab + a_split + (uint64_t)((qi * 16 + 2 * s * E::A_LBO) >> 4),
                              b0 + b_split + (uint64_t)((qi * E::B_BYTES + 2 * s * B_LBO) >> 4), acc);
              acc = 1;
            }
          }
        }
        mma_commit(&mma_done[buf]);
      }
    }
  } else {
    // ================= converters + epilogue (warps 0..7)
    auto epilogue = [&](int64_t jj) {
      const int buf = (int)(jj & 1);
      mbar_wait(&mma_done[buf], (uint32_t)((jj >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const Tile tt = tile_of(first + jj * step, tiles_per_row);
      const int quarter = warp & 3, grp = warp >> 2;       // TMEM lanes 32*quarter.., columns 8*grp..
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(buf * BLK + 8 * grp);
      float v[8];
      tmem_ld8(taddr, v);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&d_empty[buf]);
      const int64_t t0 = tt.ts + (int64_t)(32 * quarter + lane) * BLK + 8 * grp;   // block tau = 32*quarter + lane
      float* o = out + tt.row * T + t0;
      if (t0 + 8 <= T) {
        *reinterpret_cast<float4*>(o) = make_float4(fmaxf(v[0], 0.f), fmaxf(v[1], 0.f), fmaxf(v[2], 0.f), fmaxf(v[3], 0.f));
        *reinterpret_cast<float4*>(o + 4) =
            make_float4(fmaxf(v[4], 0.f), fmaxf(v[5], 0.f), fmaxf(v[6], 0.f), fmaxf(v[7], 0.f));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (t0 + i < T) o[i] = fmaxf(v[i], 0.f);
      }
    };
    for (int64_t jj = 0; jj < my_tiles; ++jj) {
      const int slot = (int)(jj % NSTAGE), buf = (int)(jj & 1);
      const Tile tt = tile_of(first + jj * step, tiles_per_row);
      mbar_wait(&stage_full[slot], (uint32_t)((jj / NSTAGE) & 1));
      if (jj >= 2) mbar_wait(&mma_done[buf], (uint32_t)(((jj - 2) >> 1) & 1));     // A[buf] no longer read
      const float* st = stage + slot * STAGE_FLOATS;
      uint8_t* a_hi = smem + E::OFF_A + (2 * buf) * E::A_BYTES;
      uint8_t* a_lo = a_hi + E::A_BYTES;
      const int64_t base_t = tt.ts - HALO * BLK;
      // one float4 (4 samples) per lane, consecutive lanes on consecutive float4s (conflict-free
      // loads); sample 4j sits in block m = j / 8 at in-block offset 4 (j % 8)
      for (int j = tid; j < STAGE_FLOATS / 4; j += THREADS) {
        const int m = j >> 3, w = j & 7;
        const int64_t t = base_t + 4 * (int64_t)j;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t >= 0 && t + 4 <= T) v = *reinterpret_cast<const float4*>(st + 4 * j);
        const float a[4] = {fabsf(v.x), fabsf(v.y), fabsf(v.z), fabsf(v.w)};
        if (BF16) {                       // half a 16-byte core row: core column w / 2, byte 8 (w % 2)
          uint32_t h[4], l[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) split<true>(a[r], h[r], l[r]);
          const uint32_t off = (uint32_t)((w >> 1) * E::A_LBO + m * 16 + (w & 1) * 8);
          *reinterpret_cast<uint2*>(a_hi + off) = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
          *reinterpret_cast<uint2*>(a_lo + off) = make_uint2(l[0] | (l[1] << 16), l[2] | (l[3] << 16));
        } else {                          // a whole 16-byte core row: core column w
          uint32_t h[4], l[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) split<false>(a[r], h[r], l[r]);
          const uint32_t off = (uint32_t)(w * E::A_LBO + m * 16);
          *reinterpret_cast<uint4*>(a_hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint4*>(a_lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
      }
      mbar_arrive(&stage_empty[slot]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a_full[buf]);
      if (jj > 0) epilogue(jj - 1);
    }
    if (my_tiles > 0) epilogue(my_tiles - 1);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
}

}  // namespace tc

cudaError_t envelope_tc_configure() {
  cudaError_t e = cudaFuncSetAttribute(tc::k_envelope_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tc::El<true>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(tc::k_envelope_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              tc::El<false>::SMEM_BYTES);
}

cudaError_t launch_envelope_tc(const float* y, float* out, int64_t rows, int64_t T, const LpTaps127& taps, int32_t L,
                               bool bf16, int sm_count, cudaStream_t st) {
  const int64_t tiles = rows * ((T + tc::TILE_T - 1) / tc::TILE_T);
  const int64_t grid = tiles < sm_count ? tiles : sm_count;
  if (bf16)
    tc::k_envelope_tc<true><<<(unsigned)grid, tc::THREADS + 64, tc::El<true>::SMEM_BYTES, st>>>(y, out, rows, T, taps, L);
  else
    tc::k_envelope_tc<false><<<(unsigned)grid, tc::THREADS + 64, tc::El<false>::SMEM_BYTES, st>>>(y, out, rows, T, taps, L);
  return cudaGetLastError();
}

}  // namespace dmas
