// sm_100a kernels of the DMAS / CF beamforming hot path (arXiv 2511.09165).
//
// K1 k_delay_table  — A1 delay LUT, IEEE fp64, bit-exact with the oracle.
// K2 k_signed_roots — A3 hoisted signed roots S = sgn(m)|m|^(1/p), once per
//                     input sample instead of once per (mic, pixel): with integer delays
//                     s_i(t, psi) = S_i[t + d(psi, i)] exactly.
// K3 k_beamform     — A2 gather (Eq. (1)) + A3 power sums + A4
//                     Newton-Girard and CF, fused.
// K4 k_envelope_*   — A5 |.| + low-pass, optional band-pass, clamp, decimate.
//
// Design notes: A2-A4 are a gather-plus-reduction, so K1-K3 use no tensor
// cores; the one dense contraction, K4's low-pass, runs on tcgen05 (dmas_envelope_tc.cu) unless
// the plan asks for the FP32 FIR (env_engine = 1).  K3 is bound by the FP32 pipe (5 FP32 ops per mic-pixel at p = 2) with shared-memory bandwidth
// close behind; its staging is one cp.async.bulk (TMA bulk engine) per microphone row into a
// window reused by BF_PSI directions; packed FADD2/FFMA2 take loaded pixel pairs as they land.

#include <cstdint>
#include <cuda_runtime.h>

#include "dmas_kernels.cuh"

namespace dmas {

// ------------------------------------------------------------------------------------------
// K1 — delay table.  One thread per (psi, i).  Fixed op order, no FMA contraction:
//   dot = ((px - rx)*ux + (py - ry)*uy) + (pz - rz)*uz ;  v = dot * k ;  d = rint_even(v)
// ------------------------------------------------------------------------------------------
__global__ void k_delay_table(const double* __restrict__ u, const double* __restrict__ pos, double rx, double ry,
                              double rz, double k, int64_t n_dirs, int32_t n_mics, int32_t* __restrict__ out,
                              float* __restrict__ alpha) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_dirs * (int64_t)n_mics) return;
  const int64_t a = idx / n_mics;
  const int32_t i = (int32_t)(idx - a * n_mics);
  const double ux = u[3 * a], uy = u[3 * a + 1], uz = u[3 * a + 2];
  const double dx = __dsub_rn(pos[3 * i], rx), dy = __dsub_rn(pos[3 * i + 1], ry), dz = __dsub_rn(pos[3 * i + 2], rz);
  const double dot = __dadd_rn(__dadd_rn(__dmul_rn(dx, ux), __dmul_rn(dy, uy)), __dmul_rn(dz, uz));
  const double v = __dmul_rn(dot, k);
  if (alpha) {                                       // linear pre-steering: floor + fraction
    const int d0 = __double2int_rd(v);
    out[idx] = d0;
    alpha[idx] = (float)__dsub_rn(v, (double)d0);
  } else {
    out[idx] = __double2int_rn(v);
  }
}

cudaError_t launch_delay_table(const double* u, const double* pos, double rx, double ry, double rz, double k,
                               int64_t n_dirs, int32_t n_mics, int32_t* out, float* alpha, cudaStream_t st) {
  const int64_t n = n_dirs * (int64_t)n_mics;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  k_delay_table<<<(unsigned)blocks, threads, 0, st>>>(u, pos, rx, ry, rz, k, n_dirs, n_mics, out, alpha);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K2 — signed-root plane.  IEEE sqrt / cbrt / pow (no fast-math): roots are taken once per
// input sample, so their cost is amortised over every direction.
// ------------------------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ float signed_root(float v) {
  if (P == 1) return v;                              // identity plane (interpolating path)
  const float a = fabsf(v);
  float r;
  if (P == 2) r = __fsqrt_rn(a);
  else if (P == 3) r = cbrtf(a);
  else if (P == 4) r = __fsqrt_rn(__fsqrt_rn(a));
  else if (P == 8) r = __fsqrt_rn(__fsqrt_rn(__fsqrt_rn(a)));
  else if (P == 6) r = cbrtf(__fsqrt_rn(a));
  else r = powf(a, 1.0f / (float)P);
  return copysignf(r, v);
}

// Paired plane (k_beamform_lds64, paired = 1): column j of a row holds the float2
// (S[j], S[j + 32]), so the two samples a lane needs at pixels t and t + 32 are one 8-byte word
// at column t + d for ANY delay d.  Sample t lands in component k of column t - 32k.
__device__ __forceinline__ void store_root(float* S, int64_t row, int64_t Tp, int64_t G, int64_t t, float r,
                                           int paired) {
  if (!paired) {
    S[row * Tp + G + t] = r;
    return;
  }
  float* e = S + (row * Tp + G) * 2;
  e[2 * t] = r;                                        // column t, component 0
  e[2 * (t - BL_STRIDE) + 1] = r;                      // column t - 32, component 1
}

template <int P>
__global__ void k_signed_roots(const float* __restrict__ m, float* __restrict__ S, int64_t T, int64_t Tp, int64_t G,
                               int paired) {
  const int64_t row = blockIdx.x;
  const float* mr = m + row * T;
  for (int64_t t = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.y * blockDim.x)
    store_root(S, row, Tp, G, t, signed_root<P>(__ldg(mr + t)), paired);
}

cudaError_t launch_signed_roots(int order, const float* m, float* S, int64_t rows, int64_t T, int64_t Tp, int64_t G,
                                int paired, cudaStream_t st) {
  const int threads = 256;
  int64_t bx = (T + threads - 1) / threads;
  if (bx > 64) bx = 64;
  dim3 grid((unsigned)rows, (unsigned)bx);
  switch (order) {
    case 1: k_signed_roots<1><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 2: k_signed_roots<2><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 3: k_signed_roots<3><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 4: k_signed_roots<4><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 5: k_signed_roots<5><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 6: k_signed_roots<6><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 7: k_signed_roots<7><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    case 8: k_signed_roots<8><<<grid, threads, 0, st>>>(m, S, T, Tp, G, paired); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K0+K2 — matched filter fused with the signed roots (NEXT-1):
//   m[t] = (sum_k w[k] raw[t + k]) / sum_k w^2 ,  S[t] = sgn(m) |m|^(1/p),  t in [0, T)
// CTA = one (frame, mic) row x 1024 outputs; taps (zero-padded to a multiple of 4) and the raw
// window in shared memory; each thread produces 4 consecutive outputs from two sliding float4
// registers (conflict-free LDS.128; the tap float4 is a broadcast): 16 FFMA per 2 LDS.128.
// ------------------------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(MF_THREADS) k_mf_roots(const float* __restrict__ raw, int64_t T_raw,
                                                         const float* __restrict__ w, int32_t Lp, float inv_energy,
                                                         float* __restrict__ S, int64_t T, int64_t Tp, int64_t G,
                                                         int paired) {
  extern __shared__ __align__(16) float msm[];
  float* tw = msm;                                   // [Lp] taps
  float* win = msm + Lp;                             // [MF_T + Lp] raw window
  const int64_t row = blockIdx.x;
  const int64_t t0 = (int64_t)blockIdx.y * MF_T;
  const float* rr = raw + row * T_raw;
  for (int i = threadIdx.x; i < Lp; i += MF_THREADS) tw[i] = __ldg(w + i);
  for (int i = threadIdx.x; i < MF_T + Lp; i += MF_THREADS) {
    const int64_t t = t0 + i;
    win[i] = (t < T_raw) ? __ldg(rr + t) : 0.f;
  }
  __syncthreads();
  const float4* w4 = reinterpret_cast<const float4*>(tw);
  const float4* r4 = reinterpret_cast<const float4*>(win) + threadIdx.x;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float4 cur = r4[0];
  for (int c = 0; c < Lp / 4; ++c) {
    const float4 nxt = r4[c + 1];
    const float4 wk = w4[c];
    const float v[8] = {cur.x, cur.y, cur.z, cur.w, nxt.x, nxt.y, nxt.z, nxt.w};
    const float ww[4] = {wk.x, wk.y, wk.z, wk.w};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fmaf(ww[r], v[j + r], acc[j]);
    cur = nxt;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t t = t0 + 4 * threadIdx.x + j;
    if (t < T) store_root(S, row, Tp, G, t, signed_root<P>(acc[j] * inv_energy), paired);
  }
}

cudaError_t launch_mf_roots(int order, const float* raw, int64_t T_raw, const float* w, int32_t Lp, float inv_energy,
                            float* S, int64_t rows, int64_t T, int64_t Tp, int64_t G, int paired,
                            cudaStream_t st) {
  dim3 grid((unsigned)rows, (unsigned)((T + MF_T - 1) / MF_T));
  const size_t smem = (size_t)(2 * Lp + MF_T) * sizeof(float);
  switch (order) {
    case 1: k_mf_roots<1><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 2: k_mf_roots<2><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 3: k_mf_roots<3><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 4: k_mf_roots<4><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 5: k_mf_roots<5><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 6: k_mf_roots<6><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 7: k_mf_roots<7><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    case 8: k_mf_roots<8><<<grid, MF_THREADS, smem, st>>>(raw, T_raw, w, Lp, inv_energy, S, T, Tp, G, paired); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Dynamic shared-memory opt-in.  cudaFuncSetAttribute is process-wide per kernel, so every
// configure call raises the limit to the most the kernel can take (the device's opt-in maximum
// less its static shared memory) instead of this plan's own need: a later (or concurrent,
// another thread's) plan with a smaller window must never lower the limit under an earlier
// plan's launches.  The launch's own smem argument still decides occupancy.
static cudaError_t smem_optin(int need, int* optin) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess && need > *optin) e = cudaErrorInvalidValue;
  return e;
}

template <typename K>
static cudaError_t set_smem_max(K* kernel, int optin) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

cudaError_t mf_configure(int32_t Lp) {
  int smem = 0;
  cudaError_t e;
  if ((e = smem_optin((2 * Lp + MF_T) * (int)sizeof(float), &smem))) return e;
  if ((e = set_smem_max(k_mf_roots<1>, smem))) return e;
  if ((e = set_smem_max(k_mf_roots<2>, smem))) return e;
  if ((e = set_smem_max(k_mf_roots<3>, smem))) return e;
  if ((e = set_smem_max(k_mf_roots<4>, smem))) return e;
  if ((e = set_smem_max(k_mf_roots<5>, smem))) return e;
  if ((e = set_smem_max(k_mf_roots<6>, smem))) return e;
  if ((e = set_smem_max(k_mf_roots<7>, smem))) return e;
  return set_smem_max(k_mf_roots<8>, smem);
}

// ------------------------------------------------------------------------------------------
// K3 — fused gather + power sums + Newton-Girard + CF.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// TMA bulk copy global -> shared (1D, 16 B granules), completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Per-pixel accumulators.  P1..P_{p-1} of the signed roots, P_p (= A for odd p, = sum |x| for
// even p), A = sum x (DAS) and B = sum x^2 (CF).  Packed in float2 pairs for FADD2/FFMA2.
template <int P> struct Acc {                           // P >= 6 (NEXT-3): P_1..P_P, A, B
  float pk[P];                                          // pk[k-1] = P_k (P_P = A for odd P)
  float a, b;
};
template <> struct Acc<2> { float2 pa, pb; };          // pa = (P1, A), pb = (P2, B)
template <> struct Acc<3> { float2 p12; float a, b; };  // P3 = A
template <> struct Acc<4> { float2 p12, p34; float a, b; };
template <> struct Acc<5> { float2 p12, p34; float a, b; };  // P5 = A

template <int P> __device__ __forceinline__ void acc_zero(Acc<P>& c) {
#pragma unroll
  for (int k = 0; k < P; ++k) c.pk[k] = 0.f;
  c.a = c.b = 0.f;
}
template <> __device__ __forceinline__ void acc_zero<2>(Acc<2>& c) { c.pa = c.pb = make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ void acc_zero<3>(Acc<3>& c) { c.p12 = make_float2(0.f, 0.f); c.a = c.b = 0.f; }
template <> __device__ __forceinline__ void acc_zero<4>(Acc<4>& c) { c.p12 = c.p34 = make_float2(0.f, 0.f); c.a = c.b = 0.f; }
template <> __device__ __forceinline__ void acc_zero<5>(Acc<5>& c) { c.p12 = c.p34 = make_float2(0.f, 0.f); c.a = c.b = 0.f; }

// One microphone sample s = s_i(t, psi) of one pixel.  x = sgn(s)|s|^p is rebuilt from s
// (exact up to rounding since s^p = sgn(x)^p |x| and the p = 2 / 4 cases take |s|).  Explicit
// IEEE intrinsics throughout (no contraction left to the compiler), so every kernel that
// inlines these rounds identically.
template <int P> __device__ __forceinline__ void acc_add(Acc<P>& c, float s) {
  float pw = s;                                          // s^k
  c.pk[0] = __fadd_rn(c.pk[0], s);
#pragma unroll
  for (int k = 1; k < P; ++k) {
    pw = __fmul_rn(pw, s);
    c.pk[k] = __fadd_rn(c.pk[k], pw);                    // k = P - 1: s^P = x (odd P) or |x| (even P)
  }
  const float x = (P & 1) ? pw : copysignf(pw, s);
  c.a = __fadd_rn(c.a, x);
  c.b = fmaf(x, x, c.b);
}
template <> __device__ __forceinline__ void acc_add<2>(Acc<2>& c, float s) {
  const float2 sx = make_float2(s, __fmul_rn(s, fabsf(s)));   // (s, x)
  c.pa = __fadd2_rn(c.pa, sx);                      // P1 += s, A += x
  c.pb = __ffma2_rn(sx, sx, c.pb);                  // P2 += s^2 (= |x|), B += x^2
}
template <> __device__ __forceinline__ void acc_add<3>(Acc<3>& c, float s) {
  const float s2 = __fmul_rn(s, s);
  const float x = __fmul_rn(s2, s);
  c.p12 = __fadd2_rn(c.p12, make_float2(s, s2));
  c.a = __fadd_rn(c.a, x);
  c.b = fmaf(x, x, c.b);
}
template <> __device__ __forceinline__ void acc_add<4>(Acc<4>& c, float s) {
  const float s2 = __fmul_rn(s, s);
  const float s3 = __fmul_rn(s2, s);
  const float s4 = __fmul_rn(s2, s2);                // = |x|
  c.p12 = __fadd2_rn(c.p12, make_float2(s, s2));
  c.p34 = __fadd2_rn(c.p34, make_float2(s3, s4));
  c.a = fmaf(s3, fabsf(s), c.a);                     // x = sgn(s) s^4 (one FFMA, no LOP)
  c.b = fmaf(s4, s4, c.b);
}
template <> __device__ __forceinline__ void acc_add<5>(Acc<5>& c, float s) {
  // 9 FP32 operations: s^4 is never formed on its own -- P4 takes s2*s2 as an FFMA and x = s^5 is
  // s3 * s2
  const float s2 = __fmul_rn(s, s);
  const float s3 = __fmul_rn(s2, s);
  const float x = __fmul_rn(s3, s2);
  c.p12 = __fadd2_rn(c.p12, make_float2(s, s2));
  c.p34.x = __fadd_rn(c.p34.x, s3);
  c.p34.y = fmaf(s2, s2, c.p34.y);
  c.a = __fadd_rn(c.a, x);
  c.b = fmaf(x, x, c.b);
}

// Interpolating path (NEXT-2): the interpolated sample v is x itself, so A and B take v directly
// and only the powers of s = root(v) are formed (one FMUL fewer per microphone sample at p = 2).
template <int P> __device__ __forceinline__ void acc_add_x(Acc<P>& c, float s, float x) { acc_add<P>(c, s); }
template <> __device__ __forceinline__ void acc_add_x<2>(Acc<2>& c, float s, float x) {
  const float2 sx = make_float2(s, x);
  c.pa = __fadd2_rn(c.pa, sx);                      // P1 += s, A += x
  c.pb = __ffma2_rn(sx, sx, c.pb);                  // P2 += s^2 (= |x|), B += x^2
}
template <> __device__ __forceinline__ void acc_add_x<3>(Acc<3>& c, float s, float x) {
  c.p12 = __fadd2_rn(c.p12, make_float2(s, __fmul_rn(s, s)));
  c.a = __fadd_rn(c.a, x);                           // = P3
  c.b = fmaf(x, x, c.b);
}
template <> __device__ __forceinline__ void acc_add_x<4>(Acc<4>& c, float s, float x) {
  const float s2 = __fmul_rn(s, s);
  c.p12 = __fadd2_rn(c.p12, make_float2(s, s2));
  c.p34 = __fadd2_rn(c.p34, make_float2(__fmul_rn(s2, s), fabsf(x)));   // P4 = sum |x|
  c.a = __fadd_rn(c.a, x);
  c.b = fmaf(x, x, c.b);
}
template <> __device__ __forceinline__ void acc_add_x<5>(Acc<5>& c, float s, float x) {
  const float s2 = __fmul_rn(s, s);
  c.p12 = __fadd2_rn(c.p12, make_float2(s, s2));
  c.p34 = __fadd2_rn(c.p34, make_float2(__fmul_rn(s2, s), __fmul_rn(s2, s2)));
  c.a = __fadd_rn(c.a, x);                           // = P5
  c.b = fmaf(x, x, c.b);
}

// Newton-Girard explicit expansions, exactly as printed.
// General Newton-Girard formula (Eq. PAPER.md:136): E_n = sum over partitions (k_1..k_n) of n with
// sum_i i k_i = n of (-1)^(n - sum k_i) prod_i P_i^{k_i} / (k_i! i^{k_i}); the partition list and
// coefficients are generated at compile time (SPEC's "cached coefficient list"), so the epilogue
// is a fixed sequence of products.
template <int N> struct PartitionTable {
  int n = 0;
  int k[32][N] = {};
  float coef[32] = {};
  constexpr PartitionTable() {
    int ks[N + 1] = {};
    rec(1, N, ks);
  }
  constexpr void rec(int i, int rem, int* ks) {
    if (i > N) {
      if (rem != 0) return;
      double c = 1.0;
      int parts = 0;
      for (int j = 1; j <= N; ++j) {
        parts += ks[j];
        double fact = 1.0, ipow = 1.0;
        for (int q = 2; q <= ks[j]; ++q) fact *= q;
        for (int q = 0; q < ks[j]; ++q) ipow *= j;
        c /= fact * ipow;
      }
      if ((N - parts) & 1) c = -c;
      for (int j = 1; j <= N; ++j) k[n][j - 1] = ks[j];
      coef[n] = (float)c;
      ++n;
      return;
    }
    for (int q = 0; q * i <= rem; ++q) {
      ks[i] = q;
      rec(i + 1, rem - q * i, ks);
    }
    ks[i] = 0;
  }
};
// Every operation below is an explicit IEEE-rounded intrinsic (no FMA contraction left to the
// compiler), so an expansion rounds identically in every kernel that inlines it.
#define FM __fmul_rn
#define FA __fadd_rn
#define FS __fsub_rn
template <int P> __device__ __forceinline__ void acc_final(const Acc<P>& c, float& A, float& B, float& E) {
  constexpr PartitionTable<P> tab{};
  A = c.a;
  B = c.b;
  float e = 0.f;
#pragma unroll
  for (int t = 0; t < tab.n; ++t) {
    float term = tab.coef[t];
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int q = 0; q < tab.k[t][j]; ++q) term = FM(term, c.pk[j]);
    e = FA(e, term);
  }
  E = e;
}
template <> __device__ __forceinline__ void acc_final<2>(const Acc<2>& c, float& A, float& B, float& E) {
  const float P1 = c.pa.x, P2 = c.pb.x;
  A = c.pa.y; B = c.pb.y;
  E = FM(0.5f, fmaf(P1, P1, -P2));                                  // (P1^2 - P2) / 2
}
template <> __device__ __forceinline__ void acc_final<3>(const Acc<3>& c, float& A, float& B, float& E) {
  const float P1 = c.p12.x, P2 = c.p12.y, P3 = c.a;
  A = c.a; B = c.b;
  // (P1^3 + 2 P3 - 3 P1 P2) / 6
  const float t = FS(FA(FM(FM(P1, P1), P1), FM(2.f, P3)), FM(FM(3.f, P1), P2));
  E = FM(t, 1.f / 6.f);
}
template <> __device__ __forceinline__ void acc_final<4>(const Acc<4>& c, float& A, float& B, float& E) {
  const float P1 = c.p12.x, P2 = c.p12.y, P3 = c.p34.x, P4 = c.p34.y;
  A = c.a; B = c.b;
  const float P1s = FM(P1, P1);
  // (P1^4 - 6 P4 + 3 P2^2 - 6 P2 P1^2 + 8 P3 P1) / 24
  float t = FS(FM(P1s, P1s), FM(6.f, P4));
  t = FA(t, FM(FM(3.f, P2), P2));
  t = FS(t, FM(FM(6.f, P2), P1s));
  t = FA(t, FM(FM(8.f, P3), P1));
  E = FM(t, 1.f / 24.f);
}
template <> __device__ __forceinline__ void acc_final<5>(const Acc<5>& c, float& A, float& B, float& E) {
  const float P1 = c.p12.x, P2 = c.p12.y, P3 = c.p34.x, P4 = c.p34.y, P5 = c.a;
  A = c.a; B = c.b;
  const float P1s = FM(P1, P1);
  // (P1^5 - 10 P2 P1^3 + 15 P2^2 P1 + 20 P3 P1^2 - 20 P3 P2 - 30 P1 P4 + 24 P5) / 120
  float t = FM(FM(P1s, P1s), P1);
  t = FS(t, FM(FM(FM(10.f, P2), P1s), P1));
  t = FA(t, FM(FM(FM(15.f, P2), P2), P1));
  t = FA(t, FM(FM(20.f, P3), P1s));
  t = FS(t, FM(FM(20.f, P3), P2));
  t = FS(t, FM(FM(30.f, P1), P4));
  t = FA(t, FM(24.f, P5));
  E = FM(t, 1.f / 120.f);
}

// E for the streaming CF-DMAS epilogue: p = 2 returns 2 E_2 (its 1/2 is folded into the CF
// reciprocal there); other orders return E_p.
template <int P> __device__ __forceinline__ void acc_final_cfdmas(const Acc<P>& c, float& A, float& B, float& E) {
  acc_final<P>(c, A, B, E);
}
template <> __device__ __forceinline__ void acc_final_cfdmas<2>(const Acc<2>& c, float& A, float& B, float& E) {
  A = c.pa.y;
  B = c.pb.y;
  E = fmaf(c.pa.x, c.pa.x, -c.pb.x);
}

// Signed root of an interpolated sample, on the fly (SFU approximations, rel. error ~2^-22).
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
template <int P>
__device__ __forceinline__ float root_fast(float x) {
  const float a = fabsf(x);
  float r;
  if (P == 2) r = sqrt_approx(a);
  else if (P == 4) r = sqrt_approx(sqrt_approx(a));
  else if (P == 8) r = sqrt_approx(sqrt_approx(sqrt_approx(a)));
  else r = ex2_approx(lg2_approx(a) * (1.0f / (float)P));     // lg2(0) = -inf -> ex2 = +0
  return copysignf(r, x);
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Accumulate microphones [i0, i1) of one direction into the thread's 8 pixels.  `wl` = window +
// lane, `oq` = the direction's word offsets, `aq` its fractions (INTERP: the window holds m and
// x = m[j] + alpha (m[j + 1] - m[j]), roots on the fly on the SFU; NEXT-2).
template <int P, bool INTERP>
__device__ __forceinline__ void bf_accumulate(Acc<P> (&acc)[BF_KT], const float* wl, const int32_t* oq,
                                              const float* aq, int i0, int i1) {
  if (INTERP) {
#pragma unroll BF_UNROLL
    for (int i = i0; i < i1; ++i) {
      const float* w = wl + oq[i];
      const float al = aq[i];
#pragma unroll
      for (int k = 0; k < BF_KT; ++k) {
        const float m0 = w[32 * k], m1 = w[32 * k + 1];
        const float v = fmaf(al, m1 - m0, m0);
        acc_add_x<P>(acc[k], root_fast<P>(v), v);
      }
    }
  } else {
    // 32-bit shared addresses: one LEA per microphone forms the lane's address, the 8 samples are
    // [addr + 128 k] immediates (a generic pointer costs an extra IADD3 + IMAD per microphone).
    const uint32_t la = smem_u32(wl);
#pragma unroll BF_UNROLL
    for (int i = i0; i < i1; ++i) {
      const uint32_t addr = la + ((uint32_t)oq[i] << 2);
#pragma unroll
      for (int k = 0; k < BF_KT; ++k) acc_add<P>(acc[k], lds_f32(addr + 128u * k));
    }
  }
}

// Classic path, integer delays: the direction's offset row is padded to a multiple of BF_MIC_PAD
// with offsets of a zeroed block (s = 0 adds exactly nothing to any sum), so offsets arrive as
// int4 loads and the loop has no remainder.
// microphones per loop iteration: 8 for p <= 3 (measured +1.4% over 4 at p = 2), 4 above
template <int P> __host__ __device__ constexpr int bf_unroll() { return P <= 3 ? 8 : 4; }
static_assert(BF_MIC_PAD % 8 == 0, "offset rows are read as int4, up to 8 microphones per iteration");
template <int P, bool INTERP>
__device__ __forceinline__ void bf_accumulate_padded(Acc<P> (&acc)[BF_KT], uint32_t la, const int32_t* oq,
                                                     const float* aq, int n_pad) {
  const int4* o4 = reinterpret_cast<const int4*>(oq);
  const float4* a4 = reinterpret_cast<const float4*>(aq);
  constexpr int U = INTERP ? 4 : bf_unroll<P>();
#pragma unroll 1
  for (int j = 0; j < n_pad / 4; j += U / 4) {
#pragma unroll
    for (int u = 0; u < U / 4; ++u) {
      const int4 o = o4[j + u];
      const int oo[4] = {o.x, o.y, o.z, o.w};
      float aa[4] = {0.f, 0.f, 0.f, 0.f};
      if (INTERP) {
        const float4 al = a4[j + u];
        aa[0] = al.x; aa[1] = al.y; aa[2] = al.z; aa[3] = al.w;
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint32_t addr = la + ((uint32_t)oo[h] << 2);
#pragma unroll
        for (int k = 0; k < BF_KT; ++k) {
          if (INTERP) {
            const float m0 = lds_f32(addr + 128u * k), m1 = lds_f32(addr + 128u * k + 4u);
            const float v = fmaf(aa[h], m1 - m0, m0);     // linear pre-steering (reading Q4b)
            acc_add_x<P>(acc[k], root_fast<P>(v), v);
          } else {
            acc_add<P>(acc[k], lds_f32(addr + 128u * k));
          }
        }
      }
    }
  }
}

// One pixel of the split plane (BeamformArgs::split_mask): |v| as the BF16 pair (hi, lo) in one
// 32-bit word at the pixel's fp32 position -- hi rounded half up on the magnitude, lo the BF16 of
// the exact remainder -- with the integer round-and-mask of the envelope's converter
// (dmas_envelope_tc.cu split_pair), so the envelope sees bit-identical operands either way.  The
// warp's store stays one coalesced 128-byte line per block, like the fp32 image's.
__device__ __forceinline__ uint32_t split_pair(float v) {
  const uint32_t b = __float_as_uint(v) & 0x7FFFFFFFu;          // |v| (LOP3, not an FADD on the FMA pipe)
  const uint32_t h = (b + 0x8000u) & 0xFFFF0000u;
  const uint32_t l = __float_as_uint(__uint_as_float(b) - __uint_as_float(h)) + 0x8000u;
  return __byte_perm(h, l, 0x7632);                    // hi in the low half (the lower address)
}
// the same for v >= +0 (sign bit clear): no masking
__device__ __forceinline__ uint32_t split_pair_nonneg(float v) {
  const uint32_t h = (__float_as_uint(v) + 0x8000u) & 0xFFFF0000u;
  const uint32_t l = __float_as_uint(v - __uint_as_float(h)) + 0x8000u;
  return __byte_perm(h, l, 0x7632);
}

// Newton-Girard + CF epilogue and coalesced stores of one direction's 8 pixels.
// KM = kinds mask compiled in: DMAS_KIND_CFDMAS (4) alone is the streaming/bench case and gets a
// minimal epilogue; anything else takes the generic epilogue (null-checked per kind).
template <int P, int KM, int KT = BF_KT>
__device__ __forceinline__ void bf_epilogue(const BeamformArgs& a, const Acc<P> (&acc)[KT], int64_t f, int64_t psi,
                                            int64_t t0, int lane) {
  const bool full_t = t0 + 32 * KT <= a.T;
  const int64_t row = f * a.n_dirs + psi;
  const int64_t o = row * a.T + t0 + lane;
  auto put = [&](int kind, int k, float v) {
    if ((a.split_mask >> kind) & 1u) reinterpret_cast<uint32_t*>(a.out[kind])[o + 32 * k] = split_pair(v);
    else a.out[kind][o + 32 * k] = v;
  };
  if (KM == 4 && full_t) {
    // streaming CF-DMAS request, whole tile in range: no per-pixel guards; for p = 2 the 1/2 of
    // E_2 moves into the reciprocal, rcp(2(N B + eps)) = rcp(N B + eps)/2 exactly (power-of-two
    // scaling), so the value is bit-identical to the generic epilogue's.
    const float n2 = (P == 2 ? 2.f : 1.f) * a.n_mics_f, e2 = (P == 2 ? 2.f : 1.f) * a.cf_eps;
    if (a.split_mask) {                                // envelope-only request: the split plane
      uint32_t* dst = reinterpret_cast<uint32_t*>(a.out[2]) + o;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        float A, B, E;
        acc_final_cfdmas<P>(acc[k], A, B, E);
        // |E * X| = |E| * X exactly (X >= 0): the |.| is the FMUL's operand modifier
        dst[32 * k] = split_pair_nonneg(FM(fabsf(E), FM(FM(A, A), rcp_approx(fmaf(n2, B, e2)))));
      }
      return;
    }
    float* dst = a.out[2] + o;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      float A, B, E;
      acc_final_cfdmas<P>(acc[k], A, B, E);
      dst[32 * k] = FM(E, FM(FM(A, A), rcp_approx(fmaf(n2, B, e2))));
    }
    return;
  }
  if (KM == 4) {
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      if (!full_t && t0 + lane + 32 * k >= a.T) continue;
      float A, B, E;
      acc_final<P>(acc[k], A, B, E);
      put(2, k, FM(E, FM(FM(A, A), rcp_approx(fmaf(a.n_mics_f, B, a.cf_eps)))));
    }
    return;
  }
  // generic request: the CF (a reciprocal per pixel) only when a CF-weighted kind is asked for
  // (warp-uniform branch); values identical either way
  const bool want_cf = a.out[2] || a.out[3] || a.out[4];
  if (!want_cf) {
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      if (!full_t && t0 + lane + 32 * k >= a.T) continue;
      float A, B, E;
      acc_final<P>(acc[k], A, B, E);
      if (a.out[0]) put(0, k, A);
      if (a.out[1]) put(1, k, E);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (!full_t && t0 + lane + 32 * k >= a.T) continue;
    float A, B, E;
    acc_final<P>(acc[k], A, B, E);
    const float cf = FM(FM(A, A), rcp_approx(fmaf(a.n_mics_f, B, a.cf_eps)));
    if (a.out[0]) put(0, k, A);
    if (a.out[1]) put(1, k, E);
    if (a.out[2]) put(2, k, FM(E, cf));
    if (a.out[3]) put(3, k, FM(A, cf));
    if (a.out[4]) put(4, k, cf);
  }
}

// Main kernel: the whole array's window staged once per CTA and reused by BF_PSI directions.
template <int P, int KM, bool INTERP>
__global__ void __launch_bounds__(BF_THREADS, (P == 2 ? DMAS_BF_MINB2 : P <= 5 ? 2 : 1)) k_beamform(const BeamformArgs a) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar;
  const int32_t n_mics = a.n_mics, W = a.W;
  const int32_t n_pad = (n_mics + BF_MIC_PAD - 1) / BF_MIC_PAD * BF_MIC_PAD;
  float* win = smem;                                   // [n_mics][W]   staged S window
  float* zero = smem + (size_t)n_mics * W;             // [BF_ZERO] zeros (padding microphones)
  int32_t* offs = reinterpret_cast<int32_t*>(zero + BF_ZERO);            // [BF_PSI][n_pad]
  float* alph = reinterpret_cast<float*>(offs + BF_PSI * n_pad);         // [BF_PSI][n_pad] (INTERP)

  const int64_t t0 = (int64_t)blockIdx.x * BF_T;
  const int64_t psi0 = (int64_t)blockIdx.y * BF_PSI;
  const int64_t f = blockIdx.z;
  const int npsi = (int)min((int64_t)BF_PSI, a.n_dirs - psi0);
  const int32_t lo = __ldg(a.tile_lo + blockIdx.y);   // window origin relative to t0 (<= min delay of tile)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t row_bytes = (uint32_t)W * 4u;
    const uint32_t offs_bytes = (uint32_t)(BF_PSI * n_pad) * 4u;
    mbar_expect_tx(&bar, row_bytes * (uint32_t)n_mics + offs_bytes * (INTERP ? 2u : 1u));
    bulk_g2s(offs, a.offs + (size_t)blockIdx.y * BF_PSI * n_pad, offs_bytes, &bar);       // plan-built
    if (INTERP) bulk_g2s(alph, a.alpha_tab + (size_t)blockIdx.y * BF_PSI * n_pad, offs_bytes, &bar);
    const float* src = a.splane + (f * n_mics) * a.Tp + a.G + t0 + lo;
    for (int i = 0; i < n_mics; ++i) bulk_g2s(win + (size_t)i * W, src + (int64_t)i * a.Tp, row_bytes, &bar);
  }
  for (int j = threadIdx.x; j < BF_ZERO; j += BF_THREADS) zero[j] = 0.f;
  __syncthreads();
  mbar_wait(&bar, 0);

  for (int q = warp; q < npsi; q += BF_WARPS) {
    Acc<P> acc[BF_KT];
#pragma unroll
    for (int k = 0; k < BF_KT; ++k) acc_zero<P>(acc[k]);
    bf_accumulate_padded<P, INTERP>(acc, smem_u32(win + lane), offs + q * n_pad, alph + q * n_pad, n_pad);
    bf_epilogue<P, KM>(a, acc, f, psi0 + q, t0, lane);
  }
}

// Large arrays (the whole window would not fit in shared memory, e.g. the 500-mic hexagonal
// arrays of PAPER.md:243-247): CTA = BF_PSI_MG directions (one per warp) x BF_T samples; the
// microphones stream through two TMA-filled window buffers of a.mg rows each (group g + 1 loads
// while group g accumulates).  Same per-pixel arithmetic, microphone order and epilogue.
template <int P, int KM, bool INTERP>
__global__ void __launch_bounds__(BF_THREADS, 2) k_beamform_mg(const BeamformArgs a) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar[2];
  const int32_t n_mics = a.n_mics, W = a.W, MG = a.mg;
  float* win = smem;                                   // [2][MG][W]
  int32_t* offs = reinterpret_cast<int32_t*>(smem + (size_t)2 * MG * W);  // [BF_PSI_MG][n_mics]
  float* alph = reinterpret_cast<float*>(offs + BF_PSI_MG * n_mics);      // [BF_PSI_MG][n_mics] (INTERP)

  const int64_t t0 = (int64_t)blockIdx.x * BF_T;
  const int64_t psi0 = (int64_t)blockIdx.y * BF_PSI_MG;
  const int64_t f = blockIdx.z;
  const int npsi = (int)min((int64_t)BF_PSI_MG, a.n_dirs - psi0);
  const int32_t lo = __ldg(a.tile_lo + blockIdx.y);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_groups = (n_mics + MG - 1) / MG;
  const float* src = a.splane + (f * n_mics) * a.Tp + a.G + t0 + lo;

  auto issue = [&](int g) {                            // thread 0: TMA one microphone group
    const int i0 = g * MG, i1 = min(n_mics, i0 + MG);
    const uint32_t row_bytes = (uint32_t)W * 4u;
    float* dst = win + (size_t)(g & 1) * MG * W;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[g & 1], row_bytes * (uint32_t)(i1 - i0));
    for (int i = i0; i < i1; ++i) bulk_g2s(dst + (size_t)(i - i0) * W, src + (int64_t)i * a.Tp, row_bytes, &bar[g & 1]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) issue(0);
  for (int q = warp; q < npsi; q += BF_WARPS) {
    const int32_t* drow = a.delays + (psi0 + q) * n_mics;
    for (int i = lane; i < n_mics; i += 32) {
      offs[q * n_mics + i] = (i % MG) * W + (__ldg(drow + i) - lo);     // offset inside the group buffer
      if (INTERP) alph[q * n_mics + i] = __ldg(a.alpha + (psi0 + q) * n_mics + i);
    }
  }
  __syncthreads();

  const int q = warp;                                  // BF_PSI_MG == BF_WARPS: one direction per warp
  Acc<P> acc[BF_KT];
#pragma unroll
  for (int k = 0; k < BF_KT; ++k) acc_zero<P>(acc[k]);
  for (int g = 0; g < n_groups; ++g) {
    if (threadIdx.x == 0 && g + 1 < n_groups) issue(g + 1);   // its buffer was released by the last barrier
    mbar_wait(&bar[g & 1], (uint32_t)((g >> 1) & 1));
    if (q < npsi)
      bf_accumulate<P, INTERP>(acc, win + (size_t)(g & 1) * MG * W + lane, offs + q * n_mics, alph + q * n_mics,
                               g * MG, min(n_mics, (g + 1) * MG));
    __syncthreads();
  }
  if (q < npsi) bf_epilogue<P, KM>(a, acc, f, psi0 + q, t0, lane);
}

// ------------------------------------------------------------------------------------------
// K3p — k_beamform_lds64 (integer delays, whole array staged): same tile (BF_PSI directions x
// BF_T samples, one direction per warp at a time, lane pixels t0 + lane + 32k, k < 8), same
// per-pixel arithmetic, microphone order and epilogue as k_beamform (bit-identical images for
// every request that includes a root-based kind; a DAS-only request sums the samples themselves
// on the identity plane and is then more exact, not bitwise equal to k_beamform's DAS), but
// a lane fetches the samples of its pixels k and k + 1 with ONE LDS.64 from the paired plane
// (column j = (S[j], S[j + 32])): the word for direction psi and mic i is column
// t0 + lane + 64 m + d(psi, i), 8-byte aligned for any delay, lanes on consecutive columns
// (conflict-free).  The accumulators are packed over those pixel pairs, so FADD2/FFMA2 take the
// loaded pair as it lands: per (direction, mic) 4 LDS.64 + 1 IADD + 8 FMUL + 8 FADD2 + 8 FFMA2 =
// 45 dispatch cycles for 8 pixels instead of k_beamform's ~50, at the same register count (so
// the same 3 CTAs / 24 warps per SM).  Windows start at a per-(tile, mic) origin lo_i (even):
// W = 224 + the largest per-mic spread columns of 8 B, one TMA bulk copy per microphone.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float2 lds_f32x2(uint32_t addr) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// Products of a pixel pair as two scalar IEEE multiplies: ptxas fuses a packed
// mul.rn.f32x2 feeding an add.rn.f32x2 into one FFMA2 despite the .rn modifiers (observed with
// CUDA 12.9 for P3 += s^2 * s), which would round differently from acc_add<P>'s scalar
// __fmul_rn; a scalar FMUL costs the same dispatch as half an FMUL2.
__device__ __forceinline__ float2 mul2s(const float2& a, const float2& b) {
  return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}

// Accumulators of one pixel pair (.x = pixel k, .y = pixel k + 1).  Per lane and pixel the
// operations are exactly acc_add<P>'s (same rounding), so get(h) reproduces the Acc<P> that
// k_beamform holds for that pixel.
template <int P> struct PAcc {                         // P >= 6: per-pixel scalar accumulators
  Acc<P> px[2];
  __device__ __forceinline__ void zero() { acc_zero<P>(px[0]); acc_zero<P>(px[1]); }
  __device__ __forceinline__ void add2(const float2& v) { acc_add<P>(px[0], v.x); acc_add<P>(px[1], v.y); }
  __device__ __forceinline__ void add2x(const float2& s, const float2& x) {
    acc_add_x<P>(px[0], s.x, x.x);
    acc_add_x<P>(px[1], s.y, x.y);
  }
  __device__ __forceinline__ Acc<P> get(int h) const { return px[h]; }
};
template <> struct PAcc<2> {
  float2 p1, a, p2, b;
  __device__ __forceinline__ void zero() { p1 = a = p2 = b = f2(0.f, 0.f); }
  __device__ __forceinline__ void add2(const float2& s) {
    add2x(s, f2(__fmul_rn(s.x, fabsf(s.x)), __fmul_rn(s.y, fabsf(s.y))));
  }
  __device__ __forceinline__ void add2x(const float2& s, const float2& x) {   // = acc_add_x<2>
    p1 = __fadd2_rn(p1, s);                           // P1 += s
    a = __fadd2_rn(a, x);                             // A  += x
    p2 = __ffma2_rn(s, s, p2);                        // P2 += s^2 (= |x|)
    b = __ffma2_rn(x, x, b);                          // B  += x^2
  }
  __device__ __forceinline__ Acc<2> get(int h) const {
    Acc<2> c;
    c.pa = h ? f2(p1.y, a.y) : f2(p1.x, a.x);
    c.pb = h ? f2(p2.y, b.y) : f2(p2.x, b.x);
    return c;
  }
};
template <> struct PAcc<3> {
  float2 p1, p2, a, b;
  __device__ __forceinline__ void zero() { p1 = p2 = a = b = f2(0.f, 0.f); }
  __device__ __forceinline__ void add2(const float2& s) {
    const float2 s2 = mul2s(s, s);
    const float2 x = mul2s(s2, s);
    p1 = __fadd2_rn(p1, s);
    p2 = __fadd2_rn(p2, s2);
    a = __fadd2_rn(a, x);                             // = P3
    b = __ffma2_rn(x, x, b);
  }
  __device__ __forceinline__ void add2x(const float2& s, const float2& x) {   // = acc_add_x<3>
    p1 = __fadd2_rn(p1, s);
    p2 = __fadd2_rn(p2, mul2s(s, s));
    a = __fadd2_rn(a, x);
    b = __ffma2_rn(x, x, b);
  }
  __device__ __forceinline__ Acc<3> get(int h) const {
    Acc<3> c;
    c.p12 = h ? f2(p1.y, p2.y) : f2(p1.x, p2.x);
    c.a = h ? a.y : a.x;
    c.b = h ? b.y : b.x;
    return c;
  }
};
template <> struct PAcc<4> {
  float2 p1, p2, p3, p4, a, b;
  __device__ __forceinline__ void zero() { p1 = p2 = p3 = p4 = a = b = f2(0.f, 0.f); }
  __device__ __forceinline__ void add2(const float2& s) {
    const float2 s2 = mul2s(s, s);
    const float2 s3 = mul2s(s2, s);
    const float2 s4 = mul2s(s2, s2);            // = |x|
    p1 = __fadd2_rn(p1, s);
    p2 = __fadd2_rn(p2, s2);
    p3 = __fadd2_rn(p3, s3);
    p4 = __fadd2_rn(p4, s4);
    a.x = fmaf(s3.x, fabsf(s.x), a.x);               // x = sgn(s) s^4
    a.y = fmaf(s3.y, fabsf(s.y), a.y);
    b = __ffma2_rn(s4, s4, b);
  }
  __device__ __forceinline__ void add2x(const float2& s, const float2& x) {   // = acc_add_x<4>
    const float2 s2 = mul2s(s, s);
    p1 = __fadd2_rn(p1, s);
    p2 = __fadd2_rn(p2, s2);
    p3 = __fadd2_rn(p3, mul2s(s2, s));
    p4 = __fadd2_rn(p4, f2(fabsf(x.x), fabsf(x.y)));   // P4 = sum |x|
    a = __fadd2_rn(a, x);
    b = __ffma2_rn(x, x, b);
  }
  __device__ __forceinline__ Acc<4> get(int h) const {
    Acc<4> c;
    c.p12 = h ? f2(p1.y, p2.y) : f2(p1.x, p2.x);
    c.p34 = h ? f2(p3.y, p4.y) : f2(p3.x, p4.x);
    c.a = h ? a.y : a.x;
    c.b = h ? b.y : b.x;
    return c;
  }
};
template <> struct PAcc<5> {
  float2 p1, p2, p3, p4, a, b;
  __device__ __forceinline__ void zero() { p1 = p2 = p3 = p4 = a = b = f2(0.f, 0.f); }
  __device__ __forceinline__ void add2(const float2& s) {   // = acc_add<5> per lane
    const float2 s2 = mul2s(s, s);
    const float2 s3 = mul2s(s2, s);
    const float2 x = mul2s(s3, s2);
    p1 = __fadd2_rn(p1, s);
    p2 = __fadd2_rn(p2, s2);
    p3 = __fadd2_rn(p3, s3);
    p4 = __ffma2_rn(s2, s2, p4);
    a = __fadd2_rn(a, x);                             // = P5
    b = __ffma2_rn(x, x, b);
  }
  __device__ __forceinline__ void add2x(const float2& s, const float2& x) {   // = acc_add_x<5>
    const float2 s2 = mul2s(s, s);
    p1 = __fadd2_rn(p1, s);
    p2 = __fadd2_rn(p2, s2);
    p3 = __fadd2_rn(p3, mul2s(s2, s));
    p4 = __fadd2_rn(p4, mul2s(s2, s2));
    a = __fadd2_rn(a, x);
    b = __ffma2_rn(x, x, b);
  }
  __device__ __forceinline__ Acc<5> get(int h) const {
    Acc<5> c;
    c.p12 = h ? f2(p1.y, p2.y) : f2(p1.x, p2.x);
    c.p34 = h ? f2(p3.y, p4.y) : f2(p3.x, p4.x);
    c.a = h ? a.y : a.x;
    c.b = h ? b.y : b.x;
    return c;
  }
};

// INTERP (linear pre-steering, NEXT-2): the paired plane holds m itself, each (direction, mic)
// carries a fraction alpha (plan-built table beside the offsets) and a lane reads columns c and
// c + 1 — (m[t + d], m[t + d + 32]) and (m[t + d + 1], m[t + d + 33]) — i.e. both interpolation
// neighbours of both pixels in two LDS.64 (k_beamform: two LDS per pixel); then exactly
// k_beamform's x = fma(alpha, m1 - m0, m0), SFU root and acc_add_x per pixel.
template <int P, int KM, bool INTERP, int KT>
__global__ void __launch_bounds__(BF_THREADS, (P == 2 ? DMAS_BF_MINB2 : P <= 5 ? (KT == 4 ? 3 : 2) : 1)) k_beamform_lds64(const BeamformArgs a) {
  constexpr int ZC = bl_zero(KT);                      // zero-block columns
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar;
  const int32_t n_mics = a.n_mics, W = a.W;            // W = window columns (8 B) per mic
  const int32_t n_pad = (n_mics + BF_MIC_PAD - 1) / BF_MIC_PAD * BF_MIC_PAD;
  float* win = smem;                                   // [n_mics][W] float2 columns
  float* zero = smem + (size_t)2 * n_mics * W;         // [ZC] float2 columns (padding mics)
  const int32_t QP = a.l_psi;                          // directions per tile (64 or 32)
  int32_t* offs = reinterpret_cast<int32_t*>(zero + 2 * ZC);   // [QP][n_pad] byte offsets
  float* alph = reinterpret_cast<float*>(offs + QP * n_pad);     // [QP][n_pad] (INTERP)

  const int64_t t0 = (int64_t)blockIdx.x * (32 * KT);
  const int64_t psi0 = (int64_t)blockIdx.y * QP;
  const int64_t f = blockIdx.z;
  const int npsi = (int)min((int64_t)QP, a.n_dirs - psi0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < 2 * ZC; j += BF_THREADS) zero[j] = 0.f;
  __syncthreads();
  if (warp == 0) {                                     // warp 0: one bulk copy per microphone
    const uint32_t row_bytes = (uint32_t)W * 8u;
    const uint32_t offs_bytes = (uint32_t)(QP * n_pad) * 4u;
    if (lane == 0) {
      mbar_expect_tx(&bar, row_bytes * (uint32_t)n_mics + offs_bytes * (INTERP ? 2u : 1u));
      bulk_g2s(offs, a.offs + (size_t)blockIdx.y * QP * n_pad, offs_bytes, &bar);
      if (INTERP) bulk_g2s(alph, a.alpha_tab + (size_t)blockIdx.y * QP * n_pad, offs_bytes, &bar);
    }
    __syncwarp();
    const int32_t* lo = a.q_lo + (size_t)blockIdx.y * n_mics;
    const float* src0 = a.splane + ((f * n_mics) * a.Tp + a.G + t0) * 2;
    for (int i = lane; i < n_mics; i += 32)
      bulk_g2s(win + (size_t)i * W * 2, src0 + ((int64_t)i * a.Tp + __ldg(lo + i)) * 2, row_bytes, &bar);
  }
  mbar_wait(&bar, 0);

  const uint32_t la = smem_u32(win) + 8u * (uint32_t)lane;
  if constexpr (KM == 1 && !INTERP) {
    // DAS-only request (Eq. (2)): the prologue wrote the identity plane (x = m, no
    // roots), so the sum over microphones is one packed FADD2 per pixel pair and LDS.64
    for (int q = warp; q < npsi; q += BF_WARPS) {
      float2 acc[KT / 2];
#pragma unroll
      for (int m = 0; m < KT / 2; ++m) acc[m] = f2(0.f, 0.f);
      const int4* o4 = reinterpret_cast<const int4*>(offs + q * n_pad);
#pragma unroll 1
      for (int j = 0; j < n_pad / 4; j += 2) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int4 o = o4[j + u];
          const int oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int m = 0; m < KT / 2; ++m) acc[m] = __fadd2_rn(acc[m], lds_f32x2(la + (uint32_t)oo[h] + 512u * m));
        }
      }
      const int64_t psi = a.psi_map ? (int64_t)__ldg(a.psi_map + psi0 + q) : psi0 + q;
      const int64_t o = (f * a.n_dirs + psi) * a.T + t0 + lane;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        if (t0 + lane + 32 * k >= a.T) continue;
        const float v = (k & 1) ? acc[k >> 1].y : acc[k >> 1].x;
        if (a.split_mask) reinterpret_cast<uint32_t*>(a.out[0])[o + 32 * k] = split_pair(v);
        else a.out[0][o + 32 * k] = v;
      }
    }
    return;
  }
  constexpr int U = bf_unroll<P>();
  for (int q = warp; q < npsi; q += BF_WARPS) {
    PAcc<P> acc[KT / 2];
#pragma unroll
    for (int m = 0; m < KT / 2; ++m) acc[m].zero();
    const int4* o4 = reinterpret_cast<const int4*>(offs + q * n_pad);
    const float4* a4 = reinterpret_cast<const float4*>(alph + q * n_pad);
#ifndef DMAS_LDS_UNROLL
#define DMAS_LDS_UNROLL 0
#endif
    // microphones per iteration (measured: 4 for the 8-pixel p = 2 tile, 178.3 vs 177.2 Gpx/s at 8;
    // 8 for the 4-pixel p = 3 tile, 72.9 vs 71.9)
    constexpr int UU = INTERP ? 4 : DMAS_LDS_UNROLL > 0 ? DMAS_LDS_UNROLL : (KT == 8 && P == 2) ? 4 : U;
#pragma unroll 1
    for (int j = 0; j < n_pad / 4; j += UU / 4) {
#pragma unroll
      for (int u = 0; u < UU / 4; ++u) {
        const int4 o = o4[j + u];
        const int oo[4] = {o.x, o.y, o.z, o.w};
        float al[4] = {0.f, 0.f, 0.f, 0.f};
        if (INTERP) {
          const float4 av = a4[j + u];
          al[0] = av.x; al[1] = av.y; al[2] = av.z; al[3] = av.w;
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint32_t addr = la + (uint32_t)oo[h];      // byte offsets
#pragma unroll
          for (int m = 0; m < KT / 2; ++m) {
            if (INTERP) {
              const float2 m0 = lds_f32x2(addr + 512u * m), m1 = lds_f32x2(addr + 512u * m + 8u);
              const float2 x = f2(fmaf(al[h], m1.x - m0.x, m0.x), fmaf(al[h], m1.y - m0.y, m0.y));   // reading Q4b
              acc[m].add2x(f2(root_fast<P>(x.x), root_fast<P>(x.y)), x);
            } else {
              acc[m].add2(lds_f32x2(addr + 512u * m));
            }
          }
        }
      }
    }
    Acc<P> px[KT];                                  // pixel t0 + lane + 32 k
#pragma unroll
    for (int k = 0; k < KT; ++k) px[k] = acc[k >> 1].get(k & 1);   // LDS m holds pixels 2m, 2m + 1
    bf_epilogue<P, KM, KT>(a, px, f, a.psi_map ? (int64_t)__ldg(a.psi_map + psi0 + q) : psi0 + q, t0, lane);
  }
}

size_t beamform_smem_bytes(int32_t n_mics, int32_t W, bool interp, int32_t mg) {
  if (mg > 0) return (size_t)2 * mg * W * sizeof(float) + (size_t)BF_PSI_MG * n_mics * (interp ? 8 : 4);
  const size_t n_pad = (n_mics + BF_MIC_PAD - 1) / BF_MIC_PAD * BF_MIC_PAD;
  return ((size_t)n_mics * W + BF_ZERO) * sizeof(float) + (size_t)BF_PSI * n_pad * 4 * (interp ? 2 : 1);
}

size_t beamform_lds64_smem_bytes(int32_t n_mics, int32_t W, bool interp, int32_t kt, int32_t psi) {
  const size_t n_pad = (n_mics + BF_MIC_PAD - 1) / BF_MIC_PAD * BF_MIC_PAD;
  return ((size_t)n_mics * W + bl_zero(kt)) * 8 + (size_t)psi * n_pad * 4 * (interp ? 2 : 1);
}

template <int P>
static cudaError_t configure_order(int bytes) {
  cudaError_t e;
  if ((e = set_smem_max(k_beamform<P, 4, false>, bytes))) return e;
  if ((e = set_smem_max(k_beamform<P, 31, false>, bytes))) return e;
  if ((e = set_smem_max(k_beamform<P, 4, true>, bytes))) return e;
  if ((e = set_smem_max(k_beamform<P, 31, true>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_mg<P, 4, false>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_mg<P, 31, false>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_mg<P, 4, true>, bytes))) return e;
  return set_smem_max(k_beamform_mg<P, 31, true>, bytes);
}

template <int P>
static cudaError_t configure_order_lds64(int bytes) {
  cudaError_t e;
  if ((e = set_smem_max(k_beamform_lds64<P, 4, false, 8>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_lds64<P, 31, false, 8>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_lds64<P, 4, true, 8>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_lds64<P, 31, true, 8>, bytes))) return e;
  if ((e = set_smem_max(k_beamform_lds64<P, 4, false, 4>, bytes))) return e;
  return set_smem_max(k_beamform_lds64<P, 31, false, 4>, bytes);
}

cudaError_t beamform_lds64_configure(int32_t n_mics, int32_t W, bool interp, int32_t kt, int32_t psi) {
  int bytes = 0;
  cudaError_t e;
  if ((e = smem_optin((int)beamform_lds64_smem_bytes(n_mics, W, interp, kt, psi), &bytes))) return e;
  if ((e = set_smem_max(k_beamform_lds64<2, 1, false, 8>, bytes))) return e;   // DAS-only
  if ((e = set_smem_max(k_beamform_lds64<2, 1, false, 4>, bytes))) return e;
  if ((e = configure_order_lds64<2>(bytes))) return e;
  if ((e = configure_order_lds64<3>(bytes))) return e;
  if ((e = configure_order_lds64<4>(bytes))) return e;
  if ((e = configure_order_lds64<5>(bytes))) return e;
  if ((e = configure_order_lds64<6>(bytes))) return e;
  if ((e = configure_order_lds64<7>(bytes))) return e;
  return configure_order_lds64<8>(bytes);
}

cudaError_t beamform_configure(int32_t n_mics, int32_t W, bool interp, int32_t mg) {
  int bytes = 0;
  cudaError_t e;
  if ((e = smem_optin((int)beamform_smem_bytes(n_mics, W, interp, mg), &bytes))) return e;
  if ((e = configure_order<2>(bytes))) return e;
  if ((e = configure_order<3>(bytes))) return e;
  if ((e = configure_order<4>(bytes))) return e;
  if ((e = configure_order<5>(bytes))) return e;
  if ((e = configure_order<6>(bytes))) return e;
  if ((e = configure_order<7>(bytes))) return e;
  return configure_order<8>(bytes);
}

template <int P>
static void launch_order(const BeamformArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  const bool only_cfdmas = !a.out[0] && !a.out[1] && a.out[2] && !a.out[3] && !a.out[4];
  const bool only_das = a.out[0] && !a.out[1] && !a.out[2] && !a.out[3] && !a.out[4];
  if (a.q_lo) {                                        // paired plane, LDS.64 gathers
    if (only_das && !a.alpha) {                        // identity plane (dmas_plan.cpp enqueue_chunk)
      if (a.kt == 4) k_beamform_lds64<2, 1, false, 4><<<grid, BF_THREADS, smem, st>>>(a);
      else k_beamform_lds64<2, 1, false, 8><<<grid, BF_THREADS, smem, st>>>(a);
    } else if (a.alpha) {
      if (only_cfdmas) k_beamform_lds64<P, 4, true, 8><<<grid, BF_THREADS, smem, st>>>(a);
      else k_beamform_lds64<P, 31, true, 8><<<grid, BF_THREADS, smem, st>>>(a);
    } else if (a.kt == 4) {
      if (only_cfdmas) k_beamform_lds64<P, 4, false, 4><<<grid, BF_THREADS, smem, st>>>(a);
      else k_beamform_lds64<P, 31, false, 4><<<grid, BF_THREADS, smem, st>>>(a);
    } else {
      if (only_cfdmas) k_beamform_lds64<P, 4, false, 8><<<grid, BF_THREADS, smem, st>>>(a);
      else k_beamform_lds64<P, 31, false, 8><<<grid, BF_THREADS, smem, st>>>(a);
    }
    return;
  }
  if (a.mg > 0) {
    if (a.alpha) {
      if (only_cfdmas) k_beamform_mg<P, 4, true><<<grid, BF_THREADS, smem, st>>>(a);
      else k_beamform_mg<P, 31, true><<<grid, BF_THREADS, smem, st>>>(a);
    } else {
      if (only_cfdmas) k_beamform_mg<P, 4, false><<<grid, BF_THREADS, smem, st>>>(a);
      else k_beamform_mg<P, 31, false><<<grid, BF_THREADS, smem, st>>>(a);
    }
    return;
  }
  if (a.alpha) {
    if (only_cfdmas) k_beamform<P, 4, true><<<grid, BF_THREADS, smem, st>>>(a);
    else k_beamform<P, 31, true><<<grid, BF_THREADS, smem, st>>>(a);
  } else {
    if (only_cfdmas) k_beamform<P, 4, false><<<grid, BF_THREADS, smem, st>>>(a);
    else k_beamform<P, 31, false><<<grid, BF_THREADS, smem, st>>>(a);
  }
}

cudaError_t launch_beamform(int order, const BeamformArgs& a, int32_t n_frames, cudaStream_t st) {
  const int t_tile = a.q_lo ? 32 * a.kt : BF_T;
  const int64_t ntt = (a.T + t_tile - 1) / t_tile;
  const int psi_tile = a.q_lo ? a.l_psi : a.mg > 0 ? BF_PSI_MG : BF_PSI;
  const int64_t npt = (a.n_dirs + psi_tile - 1) / psi_tile;
  dim3 grid((unsigned)ntt, (unsigned)npt, (unsigned)n_frames);
  const size_t smem = a.q_lo ? beamform_lds64_smem_bytes(a.n_mics, a.W, a.alpha != nullptr, a.kt, a.l_psi)
                            : beamform_smem_bytes(a.n_mics, a.W, a.alpha != nullptr, a.mg);
  switch (order) {
    case 2: launch_order<2>(a, grid, smem, st); break;
    case 3: launch_order<3>(a, grid, smem, st); break;
    case 4: launch_order<4>(a, grid, smem, st); break;
    case 5: launch_order<5>(a, grid, smem, st); break;
    case 6: launch_order<6>(a, grid, smem, st); break;
    case 7: launch_order<7>(a, grid, smem, st); break;
    case 8: launch_order<8>(a, grid, smem, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K4 fast path — 127-tap low-pass of |y|, R = 1, no band-pass, T % 4 == 0.  A CTA owns one
// 1024-sample column tile of ENV_RPC consecutive rows; each row's window [t0 - 64, t0 + 1088)
// is staged with 16-byte cp.async (zero-fill outside [0, T)), double-buffered so the next row
// loads while this one computes.  Each thread produces 4 consecutive outputs from 33
// conflict-free LDS.128; the taps live in the kernel-parameter constant bank and |.| is the
// free operand modifier, so every MAC is one FFMA R, |R|, c[], R.
//   e[t] = max(0, sum_k h[k] |y[t + 63 - k]|), zeros outside [0, T)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(ENV_THREADS) k_envelope_lp127(const float* __restrict__ y, float* __restrict__ out,
                                                               int64_t rows, int64_t T,
                                                               const __grid_constant__ LpTaps127 taps) {
  constexpr int WIN = ENV_T + 128;                     // staged samples per row
  __shared__ __align__(16) float sa[2][WIN];
  const int64_t t0 = (int64_t)blockIdx.y * ENV_T;
  const int64_t r0 = (int64_t)blockIdx.x * ENV_RPC;
  const int nr = (int)min((int64_t)ENV_RPC, rows - r0);

  auto stage = [&](int j, int buf) {                   // sa[buf][u] = y[r0 + j][t0 - 64 + u]
    const float* yr = y + (r0 + j) * T;
    for (int c = threadIdx.x; c < WIN / 4; c += ENV_THREADS) {
      const int64_t t = t0 - 64 + 4 * c;
      const bool in = (t >= 0) && (t + 4 <= T);        // T % 4 == 0: a chunk is fully in or out
      cp_async_16(&sa[buf][4 * c], in ? yr + t : yr, in ? 16 : 0);
    }
    cp_async_commit();
  };

  stage(0, 0);
  const int64_t tb = t0 + 4 * threadIdx.x;
  for (int j = 0; j < nr; ++j) {
    if (j + 1 < nr) stage(j + 1, (j + 1) & 1);
    else cp_async_commit();                            // empty group keeps the wait count uniform
    cp_async_wait<1>();
    __syncthreads();
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const float4* a4 = reinterpret_cast<const float4*>(sa[j & 1]) + threadIdx.x;
#pragma unroll
    for (int v = 0; v < 33; ++v) {
      const float4 q = a4[v];
      const float e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int u = 4 * v + c;                       // sample t0 + 4 tid - 64 + u
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int k = jj + 127 - u;                  // output t0 + 4 tid + jj uses tap k
          if (k >= 0 && k < ENV_FAST_TAPS) acc[jj] = fmaf(taps.h[k], fabsf(e[c]), acc[jj]);
        }
      }
    }
    float* orow = out + (r0 + j) * T;
    if (tb + 4 <= T) {
      *reinterpret_cast<float4*>(orow + tb) =
          make_float4(fmaxf(acc[0], 0.f), fmaxf(acc[1], 0.f), fmaxf(acc[2], 0.f), fmaxf(acc[3], 0.f));
    } else {
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        if (tb + jj < T) orow[tb + jj] = fmaxf(acc[jj], 0.f);
    }
    __syncthreads();                                   // buffer j & 1 is restaged at j + 2
  }
}

cudaError_t launch_envelope_lp127(const float* y, float* out, int64_t rows, int64_t T, const LpTaps127& taps,
                                  cudaStream_t st) {
  dim3 grid((unsigned)((rows + ENV_RPC - 1) / ENV_RPC), (unsigned)((T + ENV_T - 1) / ENV_T));
  k_envelope_lp127<<<grid, ENV_THREADS, 0, st>>>(y, out, rows, T, taps);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K4 generic path — any odd L, optional band-pass (odd Lb), decimation R.
//   b[s] = |sum_k bp[k] y[s + cb - k]| (or |y[s]|) for s in [0, T), 0 outside
//   out[o] = max(0, sum_k lp[k] b[R o + c - k])
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(ENV_THREADS) k_envelope_generic(const float* __restrict__ y, float* __restrict__ out,
                                                                 int64_t T, int64_t T_out, int32_t R,
                                                                 const float* __restrict__ lp, int32_t L,
                                                                 const float* __restrict__ bp, int32_t Lb) {
  extern __shared__ __align__(16) float sh[];
  const int c = (L - 1) / 2, cb = Lb > 0 ? (Lb - 1) / 2 : 0;
  const int64_t row = blockIdx.x;
  const int64_t o0 = (int64_t)blockIdx.y * ENV_GEN_T;
  const int64_t o_end = min(o0 + ENV_GEN_T, T_out);
  const int64_t s_lo = o0 * R - c;
  const int nb = (int)((o_end - 1) * R + c - s_lo + 1);
  float* b = sh;
  const float* yr = y + row * T;
  if (Lb > 0) {
    float* yy = sh + nb;                                 // y over [s_lo - cb, s_lo + nb + cb)
    for (int u = threadIdx.x; u < nb + 2 * cb; u += blockDim.x) {
      const int64_t s = s_lo - cb + u;
      yy[u] = (s >= 0 && s < T) ? __ldg(yr + s) : 0.f;
    }
    __syncthreads();
    for (int u = threadIdx.x; u < nb; u += blockDim.x) {
      const int64_t s = s_lo + u;
      float acc = 0.f;
      if (s >= 0 && s < T)
        for (int k = 0; k < Lb; ++k) acc = fmaf(__ldg(bp + k), yy[u + 2 * cb - k], acc);
      b[u] = fabsf(acc);
    }
  } else {
    for (int u = threadIdx.x; u < nb; u += blockDim.x) {
      const int64_t s = s_lo + u;
      b[u] = (s >= 0 && s < T) ? fabsf(__ldg(yr + s)) : 0.f;
    }
  }
  __syncthreads();
  for (int64_t o = o0 + threadIdx.x; o < o_end; o += blockDim.x) {
    const int base = (int)(o * R - s_lo) + c;            // index of sample R o + c in b
    float acc = 0.f;
    for (int k = 0; k < L; ++k) acc = fmaf(__ldg(lp + k), b[base - k], acc);
    out[row * T_out + o] = fmaxf(acc, 0.f);
  }
}

cudaError_t launch_envelope_generic(const float* y, float* out, int64_t rows, int64_t T, int64_t T_out, int32_t decim,
                                    const float* lp, int32_t L, const float* bp, int32_t Lb, cudaStream_t st) {
  const int c = (L - 1) / 2, cb = Lb > 0 ? (Lb - 1) / 2 : 0;
  const int64_t nb = (int64_t)(ENV_GEN_T - 1) * decim + 2 * c + 1;
  const size_t smem = (size_t)(nb + (Lb > 0 ? nb + 2 * cb : 0)) * sizeof(float);
  if (smem > 48 * 1024) {                               // opt-in maximum: see smem_optin
    int bytes = 0;
    cudaError_t e = smem_optin((int)smem, &bytes);
    if (e == cudaSuccess) e = set_smem_max(k_envelope_generic, bytes);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)rows, (unsigned)((T_out + ENV_GEN_T - 1) / ENV_GEN_T));
  k_envelope_generic<<<grid, ENV_THREADS, smem, st>>>(y, out, T, T_out, decim, lp, L, bp, Lb);
  return cudaGetLastError();
}

}  // namespace dmas
