// Internal launcher interface between the plan runtime (dmas_plan.cpp) and the sm_100a kernels
// (dmas_kernels.cu).  Not part of the public ABI (include/dmas.h is).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dmas {

// Beamform CTA tile (K3): BF_PSI directions x BF_T samples; 8 warps, lanes over t, 8 t / lane.
#ifndef DMAS_BF_KT
#define DMAS_BF_KT 8
#endif
#ifndef DMAS_BF_PSI
#define DMAS_BF_PSI 32
#endif
#ifndef DMAS_BF_UNROLL
#define DMAS_BF_UNROLL 2
#endif
#ifndef DMAS_BF_MINB2
#define DMAS_BF_MINB2 3
#endif
constexpr int BF_THREADS = 256;
constexpr int BF_WARPS = BF_THREADS / 32;
constexpr int BF_KT = DMAS_BF_KT;
constexpr int BF_T = 32 * BF_KT;
constexpr int BF_PSI = DMAS_BF_PSI;
constexpr int BF_UNROLL = DMAS_BF_UNROLL;   // interpolating / large-array paths
constexpr int BF_MIC_PAD = 8;              // classic path: offset rows padded to 8 microphones
constexpr int BF_ZERO = 32 * 8 + 4;        // zero block for padding microphones (+1 sample read when interpolating)
constexpr int BF_PSI_MG = BF_WARPS;     // large-array path: one direction per warp
// LDS.64 path (k_beamform_lds64): paired plane column j = (S[j], S[j + BL_STRIDE]); a lane's
// pixels k, k + 1 (t0 + lane + 32k) come from one column; the zero block covers the columns a
// padding microphone's reads span (lanes 0..31 + 64 m, m < BF_KT / 2).
constexpr int BL_STRIDE = 32;
// kt = pixels per lane (8: 256-sample tiles; 4: 128-sample tiles for arrays whose 8-pixel windows
// would not fit the CTAs per SM, e.g. 64 microphones)
__host__ __device__ constexpr int bl_span(int kt) { return 32 + 64 * (kt / 2 - 1); }   // window columns at 0 spread
__host__ __device__ constexpr int bl_zero(int kt) { return bl_span(kt) + 2; }   // (+1 read when interpolating, +1 for 16 B)

// Envelope CTA tile (K4 fast path): 1024 outputs of one row, 4 consecutive outputs / thread.
constexpr int ENV_THREADS = 256;
constexpr int ENV_T = 1024;
constexpr int ENV_FAST_TAPS = 127;
constexpr int ENV_RPC = 8;              // rows per CTA (double-buffered staging)
constexpr int ENV_GEN_T = 256;          // generic path: outputs per CTA

// Matched filter + roots (K0+K2): 1024 outputs of one (frame, mic) row per CTA, 4 per thread.
constexpr int MF_THREADS = 256;
constexpr int MF_T = 1024;
constexpr int MF_MAX_TAPS = 16384;

constexpr int N_KINDS = 5;              // DAS, DMAS, CFDMAS, CFDAS, CF (dmas.h bit order)

struct BeamformArgs {
  const float* splane;      // [frames][n_mics][Tp]; sample t of (f, i) at column G + t; zero guards
  const int32_t* delays;    // [n_dirs][n_mics] int32 sample delays d[psi][i]
  const int32_t* tile_lo;   // [n_psi_tiles] window origin (relative to t0) of each psi tile, %4 == 0
  const int32_t* offs;      // classic path: [n_psi_tiles][BF_PSI][n_pad] window word offsets i W + d - lo
                            // (padding microphones -> the zero block), built at plan time
  const float* alpha_tab;   // classic interpolating path: [n_psi_tiles][BF_PSI][n_pad] fractions (pad 0)
  float* out[N_KINDS];      // raw-image destinations [frames][n_dirs][T] (nullptr = kind not written)
  const float* alpha;       // [n_dirs][n_mics] fractional delays in [0, 1) (linear pre-steering), or null
  int32_t mg;               // > 0: large-array path, microphones staged in groups of mg (tiles of BF_PSI_MG)
  int64_t Tp, G, T, n_dirs;
  int32_t n_mics, W;        // W = staged samples per mic row (multiple of 4); LDS.64 path: columns
  float n_mics_f, cf_eps;
  // LDS.64 path (q_lo != nullptr): splane is the paired plane [frames][n_mics][Tp][2] (column
  // G + j holds (S[j], S[j + 32])); q_lo = per-(psi tile, mic) window origins in columns relative
  // to t0 (even); offs = byte offsets 8 (i W + d - lo)
  const int32_t* q_lo;      // [n_psi_tiles][n_mics]
  const int32_t* psi_map;   // LDS.64 path: tile slot psi0 + q -> image row (k-d tiles), or null (identity)
  int32_t kt;               // LDS.64 path: pixels per lane (8 or 4; 4 only without interpolation)
  int32_t l_psi;            // LDS.64 path: directions per tile (64 or 32)
  // kinds (bit k) whose out[k] is not an fp32 image but the tensor-core envelope's input: |y| as
  // the BF16 pair (hi, lo) in one 32-bit word per pixel (hi in the low half), same layout and size
  // as the fp32 image.  The split is the envelope converter's (dmas_envelope_tc.cu split_pair).
  uint32_t split_mask;
};

struct LpTaps127 { float h[128]; };

// K1: d[psi][i] = rint_even(((p_i - r) . u_psi) * k) in IEEE fp64, no contraction (A1).
// With `alpha` non-null (linear pre-steering, NEXT-2): d = floor(v) and alpha = v - d (fp32).
cudaError_t launch_delay_table(const double* u /*[n_dirs][3]*/, const double* pos /*[n_mics][3]*/,
                               double rx, double ry, double rz, double k, int64_t n_dirs, int32_t n_mics,
                               int32_t* out, float* alpha, cudaStream_t st);

// K2: S[f][i][G + t] = sgn(m) |m|^(1/p) for t in [0, T) (hoisted signed roots, A3); order 1 =
// identity (the plane of m itself, used by the interpolating beamformer).
// paired = 1 (LDS.64 beamform path): S is the paired plane [rows][Tp][2], sample t stored at
// column G + t (component 0) and column G + t - 32 (component 1); G >= 32.
cudaError_t launch_signed_roots(int order, const float* m, float* S, int64_t rows, int64_t T, int64_t Tp,
                                int64_t G, int paired, cudaStream_t st);

// K0+K2: matched filter (correlation with the zero-padded chirp w[Lp], / energy) fused with the
// signed roots; raw rows [rows][T_raw], T_raw >= T + L - 1 (NEXT-1).
cudaError_t launch_mf_roots(int order, const float* raw, int64_t T_raw, const float* w, int32_t Lp, float inv_energy,
                            float* S, int64_t rows, int64_t T, int64_t Tp, int64_t G, int paired,
                            cudaStream_t st);
cudaError_t mf_configure(int32_t Lp);

// K3: gather + power sums + Newton-Girard + CF (A2-A4).  grid = (t tiles, psi tiles, frames).
cudaError_t launch_beamform(int order, const BeamformArgs& a, int32_t n_frames, cudaStream_t st);
size_t beamform_smem_bytes(int32_t n_mics, int32_t W, bool interp, int32_t mg);
size_t beamform_lds64_smem_bytes(int32_t n_mics, int32_t W, bool interp, int32_t kt, int32_t psi);
cudaError_t beamform_lds64_configure(int32_t n_mics, int32_t W, bool interp, int32_t kt, int32_t psi);
cudaError_t beamform_configure(int32_t n_mics, int32_t W, bool interp, int32_t mg);   // > 48 KB dynamic smem

// K4: [band-pass] -> |.| -> low-pass -> clamp >= 0 -> decimate (A5), one row per (frame, psi).
cudaError_t launch_envelope_lp127(const float* y, float* out, int64_t rows, int64_t T, const LpTaps127& taps,
                                  cudaStream_t st);
// K4 tensor-core path (dmas_envelope_tc.cu): odd L <= 127, R = 1, no band-pass, T % 32 == 0,
// 16-byte aligned buffers.  Persistent: one CTA per SM.
bool envelope_tc_supported(int64_t T);
cudaError_t envelope_tc_configure();
// The constant Toeplitz tap blocks of the tensor-core envelope, built once per plan on the device
// (b_image: envelope_tc_b_bytes() bytes, 16-byte aligned); every launch bulk-copies them into
// shared memory instead of rebuilding them per CTA.
size_t envelope_tc_b_bytes();
cudaError_t envelope_tc_prepare(const LpTaps127& taps, int32_t L, void* b_image);
// out_rows_per_frame > 0: `out` rows are written as [rows / out_rows_per_frame frames][out_rows_per_frame]
// with frames out_frame_rows rows apart (a sharded plan's fused gather into the root's image).
cudaError_t launch_envelope_tc(const float* y, float* out, int64_t rows, int64_t T, const void* b_image,
                               int sm_count, cudaStream_t st, int64_t out_rows_per_frame = 0,
                               int64_t out_frame_rows = 0);
// The same on a pre-split input (BeamformArgs::split_mask layout): no converter stage.
cudaError_t launch_envelope_tc_split(const uint32_t* ysplit, float* out, int64_t rows, int64_t T, const void* b_image,
                                     int sm_count, cudaStream_t st, int64_t out_rows_per_frame = 0,
                                     int64_t out_frame_rows = 0);
cudaError_t launch_envelope_generic(const float* y, float* out, int64_t rows, int64_t T, int64_t T_out,
                                    int32_t decim, const float* lp, int32_t L, const float* bp, int32_t Lb,
                                    cudaStream_t st);

}  // namespace dmas
