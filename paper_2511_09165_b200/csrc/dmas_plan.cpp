// Host runtime behind include/dmas.h: plan validation and construction, per-call chunking,
// the host-buffer copy/compute pipeline, per-kernel event timing, error reporting.
//
// Compiled with -ffp-contract=off: the unit vectors u(psi) (A1) must round exactly like the
// oracle's Python `math` expression  (cos(el)*cos(az), cos(el)*sin(az), sin(el)).

#include "dmas.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "dmas_comm.h"
#include "dmas_kernels.cuh"

namespace {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

dmas_status fail(dmas_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                             \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      return fail(e_ == cudaErrorMemoryAllocation ? DMAS_ERR_OOM : DMAS_ERR_CUDA,                  \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                             \
    }                                                                                              \
  } while (0)

enum { K_DELAY = 0, K_ROOTS = 1, K_BEAMFORM = 2, K_ENVELOPE = 3 };

struct TimingRec {
  int kernel;
  cudaEvent_t ev0, ev1;
};

// NVTX range around a host-side enqueue step (SURVEY.md §5 tracing): visible in Nsight Systems /
// ncu --nvtx; a no-op without a tool attached.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int popcount5(uint32_t k) {
  int n = 0;
  for (int b = 0; b < dmas::N_KINDS; ++b) n += (k >> b) & 1u;
  return n;
}

}  // namespace

struct dmas_plan_s {
  std::mutex mu;
  int device = 0;
  int32_t n_mics = 0, order = 2, lp_taps = 0, bp_taps = 0, env_decim = 1, max_frames = 1;
  int64_t n_dirs = 0, T = 0, T_out = 0;
  int64_t T_in = 0;                   // input samples per channel: T, or T + mf_taps - 1 (raw)
  int32_t mf_taps = 0, mf_lp = 0;     // matched filter taps / padded to a multiple of 4
  float mf_inv_energy = 0.f;
  float* d_mf = nullptr;
  bool interp = false;                // linear-interpolation pre-steering (NEXT-2)
  float* d_alpha = nullptr;           // [n_dirs][n_mics] fractional delays
  std::vector<float> h_alpha;
  double fs = 0, c = 0;
  float cf_eps = 1e-30f;
  int32_t dmin = 0, dmax = 0;
  std::vector<int32_t> h_delays;      // [n_dirs][n_mics]
  std::vector<float> h_lp, h_bp;
  dmas::LpTaps127 lp127{};
  bool lp_fast = false;               // FP32 FIR fast path (127 taps, R = 1, no band-pass)
  bool lp_tc = false;                 // tensor-core low-pass (L <= 127, R = 1, no band-pass)
  int32_t env_engine = 0;             // 0 auto (tensor cores, BF16 split), 1 FP32 FIR, 2 tensor cores on fp32 input
  bool presplit = false;              // envelope-only kinds: the beamform writes the BF16 split plane
  int sm_count = 148;

  // device state
  int32_t* d_delays = nullptr;
  int32_t* d_tile_lo = nullptr;
  int32_t* d_offs = nullptr;          // classic path: per-tile padded window offsets
  float* d_alpha_tab = nullptr;       // classic interpolating path: per-tile padded fractions
  int32_t W = 0;                      // staged window per mic (beamform)
  int32_t mg = 0;                     // > 0: large-array path, microphones per staged group
  int32_t paired = 0;                 // LDS.64 path: paired root plane, per-(tile, mic) windows
  int32_t lds_kt = 8;                 // LDS.64 path: pixels per lane (8: 256-sample tiles, 4: 128)
  int32_t lds_psi = 32;               // LDS.64 path: directions per tile (64 or 32)
  int32_t* d_qlo = nullptr;           // LDS.64 path: [n_psi_tiles][n_mics] window origins (columns)
  int32_t* d_psi_map = nullptr;       // LDS.64 path: tile slot -> image row (k-d tiles), or null
  int64_t Tp = 0, G = 0;              // signed-root plane row length / left guard
  int32_t chunk_cap = 1;              // frames the signed-root plane holds
  float* d_splane = nullptr;
  float* d_lp = nullptr;
  void* d_tcb = nullptr;              // tensor-core envelope: the tap blocks (dmas_kernels.cuh envelope_tc_prepare)
  float* d_bp = nullptr;
  float* d_scratch = nullptr;         // raw images of envelope-only kinds
  size_t scratch_cap = 0;
  int64_t scratch_budget = 0;

  // host pipeline buffers (dmas_beamform_host), created on first use and kept
  cudaStream_t hs[3] = {nullptr, nullptr, nullptr};  // h2d, compute, d2h
  float* d_hsig[2] = {nullptr, nullptr};
  float* d_hout[2] = {nullptr, nullptr};
  size_t hsig_cap = 0, hout_cap = 0;
  cudaEvent_t h_ev[3][2] = {};                       // h2d_done, comp_done, d2h_done per buffer

  // cross-stream ordering: every call's work waits for the previous call's (the signed-root plane
  // and the scratch are shared by all calls on this plan), whatever stream either was issued on
  cudaEvent_t ev_last = nullptr;
  bool ev_last_recorded = false;

  // direction sharding over ranks; single-GPU plans: comm == nullptr
  dmas::comm::Comm* comm = nullptr;
  int32_t n_ranks = 1, rank = 0, root = 0;
  int64_t n_dirs_total = 0, dir0 = 0, n_local_max = 0;
  int32_t x_chunk_cap = 1;            // frames per exchange chunk: the minimum over ranks
  size_t x_scratch_cap = 0;           // envelope scratch: the minimum over ranks
  cudaStream_t cs = nullptr;          // comm stream: broadcasts and gathers, in one fixed order
  cudaEvent_t ev_b[2] = {}, ev_c[2] = {}, ev_g[2] = {}, ev_x0 = nullptr, ev_x1 = nullptr;
  float* d_gst[2] = {nullptr, nullptr};   // gather staging (the rank's shard of one chunk)
  size_t gst_cap = 0;
  bool status_exchanged = false;      // plan-time allreduce done (bail must not join it again)
  bool fused_gather = false;          // DMAS_GATHER of tensor-core envelopes: store into the root's image

  // timing
  bool timing = false;
  std::vector<TimingRec> recs;
  std::vector<cudaEvent_t> ev_pool;

  cudaEvent_t get_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {

// Timed launch helper: records an event pair around `fn` when the plan's timing is on.
template <class F>
cudaError_t timed(dmas_plan_s* p, int kernel, cudaStream_t st, F&& fn) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->timing) {
    e0 = p->get_event();
    e1 = p->get_event();
    cudaEventRecord(e0, st);
  }
  cudaError_t e = fn();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (p->timing) {
    cudaEventRecord(e1, st);
    p->recs.push_back({kernel, e0, e1});
  }
  return e;
}

void free_plan_memory(dmas_plan_s* p) {
  cudaFree(p->d_delays);
  cudaFree(p->d_tile_lo);
  cudaFree(p->d_qlo);
  cudaFree(p->d_psi_map);
  cudaFree(p->d_offs);
  cudaFree(p->d_alpha_tab);
  cudaFree(p->d_splane);
  cudaFree(p->d_lp);
  cudaFree(p->d_tcb);
  cudaFree(p->d_bp);
  cudaFree(p->d_mf);
  cudaFree(p->d_alpha);
  cudaFree(p->d_scratch);
  for (int b = 0; b < 2; ++b) {
    cudaFree(p->d_hsig[b]);
    cudaFree(p->d_hout[b]);
  }
  for (auto& s : p->hs)
    if (s) cudaStreamDestroy(s);
  for (auto& row : p->h_ev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  if (p->ev_last) cudaEventDestroy(p->ev_last);
  for (int b = 0; b < 2; ++b) {
    for (cudaEvent_t e : {p->ev_b[b], p->ev_c[b], p->ev_g[b]})
      if (e) cudaEventDestroy(e);
    cudaFree(p->d_gst[b]);
  }
  for (cudaEvent_t e : {p->ev_x0, p->ev_x1})
    if (e) cudaEventDestroy(e);
  if (p->cs) cudaStreamDestroy(p->cs);
  dmas::comm::destroy(p->comm);
  p->comm = nullptr;

  for (auto& r : p->recs) {
    cudaEventDestroy(r.ev0);
    cudaEventDestroy(r.ev1);
  }
  for (auto e : p->ev_pool) cudaEventDestroy(e);
}

// Blackman-windowed sinc low-pass, unit DC gain (reading Q11):
// h[n] = (2fc/fs) sinc((2fc/fs)(n - (L-1)/2)) w[n], w = 0.42 - 0.5cos(2 pi n/(L-1)) + 0.08cos(4 pi n/(L-1))
std::vector<double> blackman_lowpass(int L, double fc, double fs) {
  std::vector<double> h(L);
  const double fcn = 2.0 * fc / fs;
  double sum = 0.0;
  for (int n = 0; n < L; ++n) {
    const double x = fcn * (n - (L - 1) / 2.0);
    const double sinc = (x == 0.0) ? 1.0 : std::sin(M_PI * x) / (M_PI * x);
    const double w = (L > 1) ? 0.42 - 0.5 * std::cos(2.0 * M_PI * n / (L - 1)) + 0.08 * std::cos(4.0 * M_PI * n / (L - 1))
                             : 1.0;
    h[n] = fcn * sinc * w;
    sum += h[n];
  }
  for (auto& v : h) v /= sum;
  return h;
}

bool finite3(const double* v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }

dmas_status validate(const dmas_plan_desc* d) {
  if (!d) return fail(DMAS_ERR_NULL, "desc is NULL");
  if (!d->mic_xyz) return fail(DMAS_ERR_NULL, "mic_xyz is NULL");
  if (!d->dir_az_el) return fail(DMAS_ERR_NULL, "dir_az_el is NULL");
  if (d->n_mics < 1) return fail(DMAS_ERR_INVALID, "n_mics < 1");
  if (d->n_dirs < 1) return fail(DMAS_ERR_INVALID, "n_dirs < 1");
  if (d->n_dirs > (int64_t)65535 * dmas::BF_PSI_MG) return fail(DMAS_ERR_INVALID, "n_dirs too large");
  if (d->n_samples < 1) return fail(DMAS_ERR_INVALID, "n_samples < 1");
  if (d->n_samples > ((int64_t)1 << 30)) return fail(DMAS_ERR_INVALID, "n_samples too large");
  if (!(d->fs_hz > 0) || !std::isfinite(d->fs_hz)) return fail(DMAS_ERR_INVALID, "fs_hz must be > 0");
  if (!(d->c_mps > 0) || !std::isfinite(d->c_mps)) return fail(DMAS_ERR_INVALID, "c_mps must be > 0");
  if (d->order < 2 || d->order > 8) return fail(DMAS_ERR_ORDER, "order must be in [2,8]");
  if (d->n_mics < d->order) return fail(DMAS_ERR_ORDER, "n_mics < order (N < n)");
  if (d->order > 5 && d->n_mics < 2 * d->order)
    return fail(DMAS_ERR_ORDER, "orders 6..8 need n_mics >= 2p (fp32 Newton-Girard cancellation)");
  if (d->max_frames < 1 || d->max_frames > 65535) return fail(DMAS_ERR_INVALID, "max_frames not in [1,65535]");
  if (!(d->cf_eps >= 0.0f) || !std::isfinite(d->cf_eps)) return fail(DMAS_ERR_INVALID, "cf_eps must be >= 0");
  if (d->lp_taps < 0 || (d->lp_taps > 0 && d->lp_taps % 2 == 0) || d->lp_taps > 4095)
    return fail(DMAS_ERR_INVALID, "lp_taps must be 0 or odd (<= 4095)");
  if (d->lp_taps > 0 && !(d->lp_cutoff_hz > 0 && d->lp_cutoff_hz < d->fs_hz / 2))
    return fail(DMAS_ERR_INVALID, "lp_cutoff_hz must be in (0, fs/2)");
  if (d->bp_taps < 0 || (d->bp_taps > 0 && d->bp_taps % 2 == 0) || d->bp_taps > 4095)
    return fail(DMAS_ERR_INVALID, "bp_taps must be 0 or odd (<= 4095)");
  if (d->bp_taps > 0 && !d->bp_coeffs) return fail(DMAS_ERR_NULL, "bp_coeffs is NULL");
  if (d->bp_taps > 0 && d->lp_taps == 0) return fail(DMAS_ERR_INVALID, "band-pass needs the envelope stage");
  if (d->env_decim < 1 || d->env_decim > 64) return fail(DMAS_ERR_INVALID, "env_decim not in [1,64]");
  if (d->scratch_bytes < 0) return fail(DMAS_ERR_INVALID, "scratch_bytes < 0");
  if (d->env_engine < 0 || d->env_engine > 2) return fail(DMAS_ERR_INVALID, "env_engine not in {0, 1, 2}");
  if (d->bf_engine < 0 || d->bf_engine > 1) return fail(DMAS_ERR_INVALID, "bf_engine not in {0, 1}");
  if (d->fused_gather < 0 || d->fused_gather > 1) return fail(DMAS_ERR_INVALID, "fused_gather not in {0, 1}");
  if (d->delay_interp < 0 || d->delay_interp > 1) return fail(DMAS_ERR_INVALID, "delay_interp not in {0, 1}");
  if (d->mf_taps < 0 || d->mf_taps > dmas::MF_MAX_TAPS) return fail(DMAS_ERR_INVALID, "mf_taps not in [0, 16384]");
  if (d->mf_taps > 0 && !d->mf_coeffs) return fail(DMAS_ERR_NULL, "mf_coeffs is NULL");
  if (d->mf_taps > 0) {
    double e = 0.0;
    for (int k = 0; k < d->mf_taps; ++k) {
      if (!std::isfinite(d->mf_coeffs[k])) return fail(DMAS_ERR_INVALID, "non-finite mf_coeffs");
      e += (double)d->mf_coeffs[k] * d->mf_coeffs[k];
    }
    if (!(e > 0.0)) return fail(DMAS_ERR_INVALID, "mf_coeffs has zero energy");
  }
  for (int i = 0; i < d->n_mics; ++i)
    if (!finite3(d->mic_xyz + 3 * i)) return fail(DMAS_ERR_INVALID, "non-finite microphone position");
  if (d->reference_xyz && !finite3(d->reference_xyz)) return fail(DMAS_ERR_INVALID, "non-finite reference");
  for (int i = 0; i < d->n_mics; ++i)
    for (int j = i + 1; j < d->n_mics; ++j) {
      const double* a = d->mic_xyz + 3 * i;
      const double* b = d->mic_xyz + 3 * j;
      if (a[0] == b[0] && a[1] == b[1] && a[2] == b[2]) return fail(DMAS_ERR_INVALID, "duplicate microphone positions");
    }
  const double tol = 1e-12;
  for (int64_t a = 0; a < d->n_dirs; ++a) {
    const double az = d->dir_az_el[2 * a], el = d->dir_az_el[2 * a + 1];
    if (!std::isfinite(az) || !std::isfinite(el)) return fail(DMAS_ERR_INVALID, "non-finite direction");
    if (az < -M_PI - tol || az > M_PI + tol) return fail(DMAS_ERR_INVALID, "azimuth not in [-pi, pi]");
    if (el < -M_PI / 2 - tol || el > M_PI / 2 + tol) return fail(DMAS_ERR_INVALID, "elevation not in [-pi/2, pi/2]");
  }
  return DMAS_OK;
}

// Enqueue one chunk of frames: roots -> beamform -> envelopes.  `sig` / `outs_raw` / `outs_env`
// already point at the chunk's first frame.
//
// `split_kinds` (a subset of the envelope-only kinds, tensor-core envelope only): raw_dst[k] is the
// plan's scratch and the beamform writes it as the envelope's BF16 hi / lo split plane
// (dmas_kernels.cuh BeamformArgs::split_mask), which the envelope reads without a converter stage.
dmas_status enqueue_chunk(dmas_plan_s* p, const float* sig, int32_t nf, float* const* raw_dst,
                          float* const* env_dst, uint32_t env_kinds, cudaStream_t st, int64_t env_frame_rows = 0,
                          uint32_t split_kinds = 0) {
  // DAS-only requests on the LDS.64 path sum the samples themselves: identity plane (order 1), no
  // roots (the kernel selects its DAS-only variant on the same condition, dmas_kernels.cu)
  Nvtx range("dmas chunk");
  const bool das_only = raw_dst[0] && !raw_dst[1] && !raw_dst[2] && !raw_dst[3] && !raw_dst[4];
  const int root_order = (p->interp || (das_only && p->paired)) ? 1 : p->order;
  if (p->mf_taps > 0) {
    CUDA_TRY(timed(p, K_ROOTS, st, [&] {
      return dmas::launch_mf_roots(root_order, sig, p->T_in, p->d_mf, p->mf_lp, p->mf_inv_energy, p->d_splane,
                                   (int64_t)nf * p->n_mics, p->T, p->Tp, p->G, p->paired, st);
    }));
  } else {
    CUDA_TRY(timed(p, K_ROOTS, st, [&] {
      return dmas::launch_signed_roots(root_order, sig, p->d_splane, (int64_t)nf * p->n_mics, p->T,
                                       p->Tp, p->G, p->paired, st);
    }));
  }
  dmas::BeamformArgs a{};
  a.splane = p->d_splane;
  a.delays = p->d_delays;
  a.tile_lo = p->d_tile_lo;
  a.offs = p->d_offs;
  a.alpha_tab = p->d_alpha_tab;
  a.alpha = p->interp ? p->d_alpha : nullptr;
  a.mg = p->mg;
  for (int k = 0; k < dmas::N_KINDS; ++k) a.out[k] = raw_dst[k];
  a.Tp = p->Tp;
  a.G = p->G;
  a.T = p->T;
  a.n_dirs = p->n_dirs;
  a.n_mics = p->n_mics;
  a.W = p->W;
  a.n_mics_f = (float)p->n_mics;
  a.cf_eps = p->cf_eps;
  a.q_lo = p->d_qlo;
  a.psi_map = p->d_psi_map;
  a.kt = p->lds_kt;
  a.l_psi = p->lds_psi;
  a.split_mask = split_kinds;
  CUDA_TRY(timed(p, K_BEAMFORM, st, [&] { return dmas::launch_beamform(p->order, a, nf, st); }));
  if (!env_kinds) return DMAS_OK;
  cudaStream_t es = st;
  const int64_t rows = (int64_t)nf * p->n_dirs;
  for (int k = 0; k < dmas::N_KINDS; ++k) {
    if (!((env_kinds >> k) & 1u)) continue;
    const float* y = raw_dst[k];
    float* o = env_dst[k];
    const bool aligned16 = ((uintptr_t)y % 16 == 0) && ((uintptr_t)o % 16 == 0);
    if (env_frame_rows > 0 && !(p->lp_tc && aligned16))
      return fail(DMAS_ERR_CUDA, "internal: fused gather without the tensor-core envelope");
    if ((split_kinds >> k) & 1u) {
      if (!(p->lp_tc && aligned16)) return fail(DMAS_ERR_CUDA, "internal: split plane without the tensor-core envelope");
      CUDA_TRY(timed(p, K_ENVELOPE, es, [&] {
        return dmas::launch_envelope_tc_split(reinterpret_cast<const uint32_t*>(y), o, rows, p->T, p->d_tcb,
                                              p->sm_count, es, env_frame_rows > 0 ? p->n_dirs : 0,
                                              env_frame_rows);
      }));
    } else if (p->lp_tc && aligned16) {
      CUDA_TRY(timed(p, K_ENVELOPE, es, [&] {
        return dmas::launch_envelope_tc(y, o, rows, p->T, p->d_tcb, p->sm_count, es,
                                        env_frame_rows > 0 ? p->n_dirs : 0, env_frame_rows);
      }));
    } else if (p->lp_fast && aligned16) {
      CUDA_TRY(timed(p, K_ENVELOPE, es, [&] { return dmas::launch_envelope_lp127(y, o, rows, p->T, p->lp127, es); }));
    } else {
      CUDA_TRY(timed(p, K_ENVELOPE, es, [&] {
        return dmas::launch_envelope_generic(y, o, rows, p->T, p->T_out, p->env_decim, p->d_lp, p->lp_taps, p->d_bp,
                                             p->bp_taps, es);
      }));
    }
  }
  return DMAS_OK;
}

dmas_status check_what(dmas_plan_s* p, uint32_t what, uint32_t& raw_k, uint32_t& env_k) {
  raw_k = what & DMAS_KIND_ALL;
  env_k = (what >> 8) & DMAS_KIND_ALL;
  if (what & ~(uint32_t)(DMAS_RAW(DMAS_KIND_ALL) | DMAS_ENV(DMAS_KIND_ALL) | DMAS_GATHER | DMAS_SIGNALS_RESIDENT))
    return fail(DMAS_ERR_SHAPE, "unknown bits in `what`");
  if (!raw_k && !env_k) return fail(DMAS_ERR_SHAPE, "`what` requests no output");
  if (env_k && p->lp_taps == 0) return fail(DMAS_ERR_SHAPE, "envelope requested on a plan without envelope stage");
  return DMAS_OK;
}

// Core of dmas_beamform on device pointers (caller holds p->mu and the device guard).
//
// Frames go through in chunks (the signed-root plane and the envelope scratch hold one chunk).
// Sharded plans add the exchange on the plan's comm stream `cs`, issued in one
// fixed order that every rank repeats (NCCL needs the same sequence on all ranks): broadcast of
// chunks 0 and 1, then per chunk c: [compute c on `st`] -> gather c -> broadcast c + 2.  The
// broadcast of chunk c + 1 thus overlaps the compute of chunk c, and the gather of chunk c the
// compute of chunk c + 1 (the shard staging is double-buffered).  The chunk size depends only on
// quantities every rank shares (allreduced at plan time), so the messages match on all ranks.
dmas_status beamform_device(dmas_plan_s* p, const float* signals, int32_t n_frames, float* const* outs,
                            uint32_t raw_k, uint32_t env_k, uint32_t flags, cudaStream_t st) {
  const bool sharded = p->comm != nullptr;
  bool gather = sharded && (flags & DMAS_GATHER);
  const bool bcast = sharded && !(flags & DMAS_SIGNALS_RESIDENT);
  const bool is_root = p->rank == p->root;
  // requested outputs in `outs` order: raw kinds, then envelope kinds, in bit order
  struct Out {
    int k;
    bool env;
    int64_t row;         // floats per image row
    float* user;         // caller's buffer (nullptr on non-root ranks when gathering)
    size_t stage_off;    // floats: offset of this output's region in a gather staging buffer
  };
  Out o[2 * dmas::N_KINDS];
  int n = 0;
  for (int k = 0; k < dmas::N_KINDS; ++k)
    if ((raw_k >> k) & 1u) o[n++] = {k, false, p->T, nullptr, 0};
  for (int k = 0; k < dmas::N_KINDS; ++k)
    if ((env_k >> k) & 1u) o[n++] = {k, true, p->T_out, nullptr, 0};
  const bool user_outs = !(gather && !is_root);
  if (user_outs && !outs) return fail(DMAS_ERR_NULL, "outs is NULL");
  for (int i = 0; i < n; ++i) {
    if (!user_outs) break;
    o[i].user = outs[i];
    if (!outs[i]) return fail(DMAS_ERR_NULL, "output pointer is NULL");
    if (((uintptr_t)outs[i]) & 3u) return fail(DMAS_ERR_SHAPE, "misaligned output pointer");
  }
  // envelope kinds without their raw image go through the plan's scratch (allocated by dmas_plan:
  // at least one frame of every kind, so a call never allocates or synchronises)
  const uint32_t env_only = env_k & ~raw_k;
  const int n_scratch = popcount5(env_only);
  const int64_t rows_sz = sharded ? p->n_local_max : p->n_dirs;     // identical on every rank
  const size_t frame_img = (size_t)rows_sz * p->T * sizeof(float);
  int32_t chunk = std::min(sharded ? p->x_chunk_cap : p->chunk_cap, n_frames);
  if (n_scratch > 0) {
    const size_t fit = (sharded ? p->x_scratch_cap : p->scratch_cap) / (frame_img * n_scratch);
    if (fit < 1) return fail(DMAS_ERR_CUDA, "internal: envelope scratch smaller than one frame");
    chunk = (int32_t)std::min<size_t>((size_t)chunk, fit);
  }
  // fused gather: an envelope-only request on the tensor-core envelope, so the last kernel of every
  // output can store its rows straight into the root's image (include/dmas.h fused_gather).  The
  // condition is the same on every rank; the root's buffers are exchanged (collectively) and every
  // rank checks the 16-byte alignment TMA needs on the pointer it received, so all ranks agree.
  bool fused = gather && p->fused_gather && raw_k == 0 && p->lp_tc && (p->T_out * sizeof(float)) % 16 == 0;
  void* mapped[2 * dmas::N_KINDS] = {};
  if (fused) {
    std::string err;
    for (int i = 0; i < n; ++i) {
      dmas_status rc = dmas::comm::map_root_buffer(p->comm, is_root ? o[i].user : nullptr, p->root, &mapped[i],
                                                   p->cs, err);
      if (rc != DMAS_OK) return fail(rc, err);
      fused = fused && ((uintptr_t)mapped[i] % 16 == 0);
    }
    if (fused) gather = false;                        // no staging, no send / recv
  }
  if (gather) {
    size_t per_frame = 0;
    for (int i = 0; i < n; ++i) per_frame += (size_t)rows_sz * o[i].row * sizeof(float);
    const size_t fit = p->gst_cap / per_frame;
    if (fit < 1) return fail(DMAS_ERR_SHAPE, "one frame of the requested images exceeds the gather staging");
    chunk = (int32_t)std::min<size_t>((size_t)chunk, fit);
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
      o[i].stage_off = off;
      off += (size_t)chunk * p->n_dirs * o[i].row;
    }
  }
  const int32_t n_chunks = (n_frames + chunk - 1) / chunk;
  // envelope-only kinds on the tensor-core envelope take the pre-split scratch (no converter pass)
  // when their envelope destination meets the 16-byte alignment TMA needs
  uint32_t split_k = 0;
  if (p->presplit)
    for (int i = 0; i < n; ++i)
      if (o[i].env && ((env_only >> o[i].k) & 1u) &&
          (fused ? (uintptr_t)mapped[i] % 16 == 0 : gather || (uintptr_t)o[i].user % 16 == 0))
        split_k |= 1u << o[i].k;
  // under CUDA-graph capture the calls are ordered by the captured stream itself, and an event
  // recorded outside the capture must not be waited on inside it
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(st, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (capturing && sharded) return fail(DMAS_ERR_SHAPE, "sharded plans cannot be captured in a CUDA graph");
  if (p->ev_last_recorded && !capturing) CUDA_TRY(cudaStreamWaitEvent(st, p->ev_last, 0));
  std::string err;
  Nvtx range(sharded ? (gather ? "dmas_beamform sharded+gather" : "dmas_beamform sharded") : "dmas_beamform");
  auto issue_bcast = [&](int32_t c) -> dmas_status {
    Nvtx r("dmas broadcast");
    const int32_t f0 = c * chunk, nf = std::min(chunk, n_frames - f0);
    float* sig = const_cast<float*>(signals) + (size_t)f0 * p->n_mics * p->T_in;
    dmas_status rc = dmas::comm::broadcast(p->comm, sig, (size_t)nf * p->n_mics * p->T_in, p->root, p->cs, err);
    if (rc != DMAS_OK) return fail(rc, err);
    CUDA_TRY(cudaEventRecord(p->ev_b[c & 1], p->cs));
    return DMAS_OK;
  };
  if (sharded) {
    CUDA_TRY(cudaEventRecord(p->ev_x0, st));
    CUDA_TRY(cudaStreamWaitEvent(p->cs, p->ev_x0, 0));
    for (int32_t c = 0; bcast && c < std::min(2, n_chunks); ++c) {
      dmas_status rc = issue_bcast(c);
      if (rc != DMAS_OK) return rc;
    }
  }
  for (int32_t c = 0; c < n_chunks; ++c) {
    const int32_t f0 = c * chunk, nf = std::min(chunk, n_frames - f0);
    if (bcast) CUDA_TRY(cudaStreamWaitEvent(st, p->ev_b[c & 1], 0));
    if (gather && c >= 2) CUDA_TRY(cudaStreamWaitEvent(st, p->ev_g[c & 1], 0));
    float* raw_dst[dmas::N_KINDS] = {};
    float* env_dst[dmas::N_KINDS] = {};
    for (int i = 0; i < n; ++i) {
      float* dst = fused    ? static_cast<float*>(mapped[i]) + ((size_t)f0 * p->n_dirs_total + p->dir0) * o[i].row
                   : gather ? p->d_gst[c & 1] + o[i].stage_off
                            : o[i].user + (size_t)f0 * p->n_dirs * o[i].row;
      (o[i].env ? env_dst : raw_dst)[o[i].k] = dst;
    }
    int s = 0;
    for (int k = 0; k < dmas::N_KINDS; ++k)
      if ((env_only >> k) & 1u) raw_dst[k] = p->d_scratch + (size_t)(s++) * chunk * p->n_dirs * p->T;
    const float* sig = signals + (size_t)f0 * p->n_mics * p->T_in;
    dmas_status rc = enqueue_chunk(p, sig, nf, raw_dst, env_dst, env_k, st, fused ? p->n_dirs_total : 0, split_k);
    if (rc != DMAS_OK) return rc;
    if (gather) {
      Nvtx r("dmas gather");
      CUDA_TRY(cudaEventRecord(p->ev_c[c & 1], st));
      CUDA_TRY(cudaStreamWaitEvent(p->cs, p->ev_c[c & 1], 0));
      for (int i = 0; i < n; ++i) {
        const std::vector<dmas_xfer> xs =
            dmas::comm::gather_schedule(p->n_dirs_total, p->n_ranks, p->rank, p->root, nf, o[i].row);
        float* dst = is_root ? o[i].user + (size_t)f0 * p->n_dirs_total * o[i].row : nullptr;
        rc = dmas::comm::run_gather(p->comm, xs, p->d_gst[c & 1] + o[i].stage_off, dst, p->cs, err);
        if (rc != DMAS_OK) return fail(rc, err);
      }
      CUDA_TRY(cudaEventRecord(p->ev_g[c & 1], p->cs));
    }
    if (bcast && c + 2 < n_chunks) {
      rc = issue_bcast(c + 2);
      if (rc != DMAS_OK) return rc;
    }
  }
  if (fused) {
    // the root's stream must not run ahead of the other ranks' stores into its images
    CUDA_TRY(cudaEventRecord(p->ev_x0, st));
    CUDA_TRY(cudaStreamWaitEvent(p->cs, p->ev_x0, 0));
    std::string err;
    dmas_status rc = dmas::comm::root_barrier(p->comm, p->root, p->cs, err);
    if (rc != DMAS_OK) return fail(rc, err);
  }
  if (sharded) {
    CUDA_TRY(cudaEventRecord(p->ev_x1, p->cs));
    CUDA_TRY(cudaStreamWaitEvent(st, p->ev_x1, 0));
  }
  if (!capturing) {
    CUDA_TRY(cudaEventRecord(p->ev_last, st));
    p->ev_last_recorded = true;
  }
  return DMAS_OK;
}

}  // namespace

extern "C" {

void dmas_plan_desc_init(dmas_plan_desc* d) {
  if (!d) return;
  std::memset(d, 0, sizeof(*d));
  d->order = 2;
  d->max_frames = 1;
  d->cf_eps = 1e-30f;
  d->lp_taps = 127;
  d->lp_cutoff_hz = 5000.0;
  d->env_decim = 1;
  d->device = -1;
}

dmas_status dmas_plan(const dmas_plan_desc* desc, dmas_plan_t* out) {
  if (!out) return fail(DMAS_ERR_NULL, "out is NULL");
  *out = nullptr;
  Nvtx range("dmas_plan");
  dmas_status st = validate(desc);
  if (st != DMAS_OK) return st;
  // direction sharding: the plan is built for this rank's contiguous slice of the
  // grid; everything below sees only the slice
  const bool sharded = desc->n_ranks > 1 || desc->comm_id != nullptr;
  const int32_t n_ranks = std::max(1, desc->n_ranks);
  int64_t g0 = 0, g1 = desc->n_dirs;
  if (sharded) {
    if (!desc->comm_id) return fail(DMAS_ERR_NULL, "comm_id is NULL (n_ranks > 1)");
    if (desc->rank < 0 || desc->rank >= n_ranks) return fail(DMAS_ERR_INVALID, "rank not in [0, n_ranks)");
    if (desc->root < 0 || desc->root >= n_ranks) return fail(DMAS_ERR_INVALID, "root not in [0, n_ranks)");
    if (desc->n_dirs < n_ranks) return fail(DMAS_ERR_INVALID, "fewer directions than ranks");
    dmas::comm::shard_range(desc->n_dirs, n_ranks, desc->rank, &g0, &g1);
  }
  dmas_plan_desc local_desc = *desc;
  local_desc.n_dirs = g1 - g0;
  local_desc.dir_az_el = desc->dir_az_el + 2 * g0;
  const dmas_plan_desc* full_desc = desc;
  desc = &local_desc;

  int dev = desc->device;
  if (dev < 0) CUDA_TRY(cudaGetDevice(&dev));
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (dev >= ndev) return fail(DMAS_ERR_INVALID, "device ordinal out of range");
  DeviceGuard guard(dev);

  auto* p = new dmas_plan_s();
  p->device = dev;
  p->n_mics = desc->n_mics;
  p->n_dirs = desc->n_dirs;
  p->n_dirs_total = full_desc->n_dirs;
  p->dir0 = g0;
  p->n_ranks = n_ranks;
  p->rank = sharded ? desc->rank : 0;
  p->root = sharded ? desc->root : 0;
  p->n_local_max = (full_desc->n_dirs + n_ranks - 1) / n_ranks;
  p->fused_gather = sharded && full_desc->fused_gather == 1;
  p->T = desc->n_samples;
  p->order = desc->order;
  p->max_frames = desc->max_frames;
  p->fs = desc->fs_hz;
  p->c = desc->c_mps;
  p->cf_eps = desc->cf_eps;
  p->lp_taps = desc->lp_taps;
  p->bp_taps = desc->bp_taps;
  p->env_decim = desc->env_decim;
  p->T_out = (p->T + p->env_decim - 1) / p->env_decim;
  p->mf_taps = desc->mf_taps;
  p->T_in = p->T + (p->mf_taps > 0 ? p->mf_taps - 1 : 0);
  p->scratch_budget = desc->scratch_bytes > 0 ? desc->scratch_bytes : ((int64_t)4 << 30);

  auto bail = [&](dmas_status s) {
    if (p->comm && !p->status_exchanged) {
      // the other ranks wait in the plan-time allreduce: contribute "failed" so they fail too
      int64_t v = 0;
      std::string ignored;
      dmas::comm::allreduce_min(p->comm, &v, p->cs, ignored);
    }
    free_plan_memory(p);
    delete p;
    return s;
  };
#define PLAN_TRY(expr)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return bail(fail(e_ == cudaErrorMemoryAllocation ? DMAS_ERR_OOM : DMAS_ERR_CUDA,            \
                       std::string(#expr) + ": " + cudaGetErrorString(e_)));                      \
  } while (0)
  if (sharded) {
    // the communicator first: every rank reaches this point (validation is identical on all), and
    // a failure further down is then reported to the others through the plan-time allreduce
    PLAN_TRY(cudaStreamCreateWithFlags(&p->cs, cudaStreamNonBlocking));
    std::string err;
    dmas_status rc = dmas::comm::create(full_desc->comm_id, n_ranks, p->rank, &p->comm, err);
    if (rc != DMAS_OK) return bail(fail(rc, err));
  }

  // ---- A1: unit vectors on the host (libm, no contraction), table on the device
  const int64_t nd = p->n_dirs;
  const int32_t nm = p->n_mics;
  std::vector<double> u((size_t)nd * 3);
  for (int64_t a = 0; a < nd; ++a) {
    const double az = desc->dir_az_el[2 * a], el = desc->dir_az_el[2 * a + 1];
    const double ce = std::cos(el);
    u[3 * a] = ce * std::cos(az);
    u[3 * a + 1] = ce * std::sin(az);
    u[3 * a + 2] = std::sin(el);
  }
  const double rx = desc->reference_xyz ? desc->reference_xyz[0] : 0.0;
  const double ry = desc->reference_xyz ? desc->reference_xyz[1] : 0.0;
  const double rz = desc->reference_xyz ? desc->reference_xyz[2] : 0.0;
  // |v| <= |p - r| fs / c must fit comfortably in int32 windows
  double rmax = 0.0;
  for (int i = 0; i < nm; ++i) {
    const double* q = desc->mic_xyz + 3 * i;
    rmax = std::max(rmax, std::sqrt((q[0] - rx) * (q[0] - rx) + (q[1] - ry) * (q[1] - ry) + (q[2] - rz) * (q[2] - rz)));
  }
  if (rmax * p->fs / p->c > 1.0e6) return bail(fail(DMAS_ERR_INVALID, "delay range exceeds 1e6 samples"));
  const double k = -(p->fs / p->c);

  double* d_u = nullptr;
  double* d_pos = nullptr;
  PLAN_TRY(cudaMalloc(&d_u, u.size() * sizeof(double)));
  PLAN_TRY(cudaMalloc(&d_pos, (size_t)nm * 3 * sizeof(double)));
  PLAN_TRY(cudaMalloc(&p->d_delays, (size_t)nd * nm * sizeof(int32_t)));
  p->interp = desc->delay_interp == 1;
  if (p->interp) PLAN_TRY(cudaMalloc(&p->d_alpha, (size_t)nd * nm * sizeof(float)));
  PLAN_TRY(cudaMemcpy(d_u, u.data(), u.size() * sizeof(double), cudaMemcpyHostToDevice));
  PLAN_TRY(cudaMemcpy(d_pos, desc->mic_xyz, (size_t)nm * 3 * sizeof(double), cudaMemcpyHostToDevice));
  PLAN_TRY(timed(p, K_DELAY, nullptr,
                 [&] { return dmas::launch_delay_table(d_u, d_pos, rx, ry, rz, k, nd, nm, p->d_delays, p->d_alpha,
                                                       nullptr); }));
  p->h_delays.resize((size_t)nd * nm);
  PLAN_TRY(cudaMemcpy(p->h_delays.data(), p->d_delays, p->h_delays.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (p->interp) {
    p->h_alpha.resize((size_t)nd * nm);
    PLAN_TRY(cudaMemcpy(p->h_alpha.data(), p->d_alpha, p->h_alpha.size() * sizeof(float), cudaMemcpyDeviceToHost));
  }
  cudaFree(d_u);
  cudaFree(d_pos);

  // ---- beamform staging metadata: per psi tile window origin (aligned down to 4) and width.
  // Classic path (whole-array window, BF_PSI directions per CTA) when it fits in <= 116 KB of
  // shared memory (2+ CTAs/SM); otherwise the large-array path streams microphone groups.
  int32_t lo_min = INT32_MAX, lo_max = INT32_MIN;
  std::vector<int32_t> tile_lo;
  auto make_tiles = [&](int psi_tile) {
    const int64_t n_pt = (nd + psi_tile - 1) / psi_tile;
    tile_lo.assign((size_t)n_pt, 0);
    p->dmin = INT32_MAX;
    p->dmax = INT32_MIN;
    lo_min = INT32_MAX;
    lo_max = INT32_MIN;
    int32_t wmax = 0;
    for (int64_t t = 0; t < n_pt; ++t) {
      int32_t lo = INT32_MAX, hi = INT32_MIN;
      const int64_t a1 = std::min<int64_t>(nd, (t + 1) * psi_tile);
      for (int64_t a = t * psi_tile; a < a1; ++a)
        for (int i = 0; i < nm; ++i) {
          const int32_t v = p->h_delays[(size_t)a * nm + i];
          lo = std::min(lo, v);
          hi = std::max(hi, v);
        }
      p->dmin = std::min(p->dmin, lo);
      p->dmax = std::max(p->dmax, hi);
      const int32_t lo_al = (int32_t)(std::floor(lo / 4.0) * 4);
      tile_lo[(size_t)t] = lo_al;
      lo_min = std::min(lo_min, lo_al);
      lo_max = std::max(lo_max, lo_al);
      wmax = std::max(wmax, dmas::BF_T + (hi - lo_al) + (p->interp ? 1 : 0));   // + m[j + 1] when interpolating
    }
    p->W = (wmax + 3) / 4 * 4;
  };
  make_tiles(dmas::BF_PSI);
  p->mg = 0;
  if (dmas::beamform_smem_bytes(nm, p->W, p->interp, 0) > (size_t)116 * 1024) {
    make_tiles(dmas::BF_PSI_MG);
    const int64_t fixed = (int64_t)dmas::BF_PSI_MG * nm * (p->interp ? 8 : 4);
    int64_t mg = ((int64_t)100 * 1024 - fixed) / (8 * (int64_t)p->W);
    mg = std::max<int64_t>(4, std::min<int64_t>(mg / 4 * 4, nm));
    p->mg = (int32_t)mg;
  }
  // LDS.64 path (k_beamform_lds64): integer delays, whole array staged, and its windows (per
  // (tile, mic) origin lo = min over the tile's directions of d, aligned down to even; W = 224 +
  // the largest per-mic spread columns of 8 B) fit as many CTAs per SM as k_beamform gets.  A
  // tile's 64 or 32 directions need not be consecutive rows: the plan also groups them by recursive
  // bisection of the unit vectors (k-d tree, splits at multiples of the tile), so a tile is a compact
  // patch of the sky even when the grid's row order makes consecutive rows far apart (e.g.
  // elevation-fastest grids whose long columns are not multiples of 32), and keeps whichever
  // order gives the narrower window; the kernel then writes each direction to its own row
  // through psi_map (the image layout is unchanged).
  const int64_t n_pad = (nm + dmas::BF_MIC_PAD - 1) / dmas::BF_MIC_PAD * dmas::BF_MIC_PAD;
  std::vector<int32_t> qlo, order;
  if (p->mg == 0 && desc->bf_engine == 0) {
    // per-(tile, mic) window origins and the largest spread for tiles of `psi` directions taken
    // in order `ord` (null = consecutive rows)
    auto eval = [&](int psi, const std::vector<int32_t>* ord, std::vector<int32_t>& lo_t, int32_t& wmax,
                    int32_t& lmin, int32_t& lmax) {
      const int64_t n_pt = (nd + psi - 1) / psi;
      lo_t.assign((size_t)n_pt * nm, 0);
      wmax = 0;
      lmin = INT32_MAX;
      lmax = INT32_MIN;
      for (int64_t t = 0; t < n_pt; ++t) {
        const int64_t a1 = std::min<int64_t>(nd, (t + 1) * psi);
        for (int i = 0; i < nm; ++i) {
          int32_t lo = INT32_MAX, hi = INT32_MIN;
          for (int64_t k = t * psi; k < a1; ++k) {
            const int64_t a = ord ? (*ord)[(size_t)k] : k;
            const int32_t v = p->h_delays[(size_t)a * nm + i];
            lo = std::min(lo, v);
            hi = std::max(hi, v);
          }
          const int32_t lo_al = (int32_t)(std::floor(lo / 2.0) * 2);
          lo_t[(size_t)t * nm + i] = lo_al;
          lmin = std::min(lmin, lo_al);
          lmax = std::max(lmax, lo_al);
          wmax = std::max(wmax, hi - lo_al);           // spread; window = bl_span(kt) + spread (+1)
        }
      }
    };
    // k-d grouping: split the set at a multiple of psi along the unit-vector component with the
    // largest range, recursively, so every tile but the last holds exactly psi directions
    auto kd_order = [&](int psi) {
      std::vector<int32_t> ord((size_t)nd);
      for (int64_t a = 0; a < nd; ++a) ord[(size_t)a] = (int32_t)a;
      const int64_t G = psi;
      std::vector<std::pair<int64_t, int64_t>> stack{{0, nd}};
      while (!stack.empty()) {
        const auto [b, e] = stack.back();
        stack.pop_back();
        const int64_t n = e - b;
        if (n <= G) continue;
        double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
        for (int64_t k = b; k < e; ++k)
          for (int c3 = 0; c3 < 3; ++c3) {
            mn[c3] = std::min(mn[c3], u[3 * (size_t)ord[k] + c3]);
            mx[c3] = std::max(mx[c3], u[3 * (size_t)ord[k] + c3]);
          }
        int ax = 0;
        for (int c3 = 1; c3 < 3; ++c3)
          if (mx[c3] - mn[c3] > mx[ax] - mn[ax]) ax = c3;
        std::sort(ord.begin() + b, ord.begin() + e, [&](int32_t x, int32_t y) {
          const double ux = u[3 * (size_t)x + ax], uy = u[3 * (size_t)y + ax];
          return ux < uy || (ux == uy && x < y);
        });
        int64_t left = std::max<int64_t>(G, (n / 2 + G / 2) / G * G);
        if (left >= n) left = G;
        stack.push_back({b + left, e});
        stack.push_back({b, b + left});
      }
      return ord;
    };
    // Pick the tile: 8 pixels per lane (256-sample tiles) when its windows fit as many CTAs per SM
    // as k_beamform gets (launch bounds: 3 at p = 2, 2 at p = 3..5, 1 above), else 4 pixels per
    // lane (128-sample tiles, 3 CTAs per SM; integer delays, p <= 5) — 64-microphone arrays (C4);
    // within a pixel count, 64 directions per tile before 32 (staging amortised over twice the
    // work: +0.3-0.5% measured), and consecutive rows before k-d tiles at equal tile size
    // (measured 1-3% faster on C5 at 32), k-d tiles when they are what makes the window fit.
    const int extra = p->interp ? 1 : 0;                 // + m[j + 1]
#ifndef DMAS_LDS_KT4_FIRST
#define DMAS_LDS_KT4_FIRST 0
#endif
    std::vector<int32_t> lo_n, lo_k, kd_ord;
    int32_t w_n = 0, w_k = 0, lmin_n = 0, lmax_n = 0, lmin_k = 0, lmax_k = 0;
    for (int kt : {DMAS_LDS_KT4_FIRST ? 4 : 8, DMAS_LDS_KT4_FIRST ? 8 : 4}) {
      if (kt == 4 && (p->interp || p->order > 5)) continue;
      const size_t budget = (p->order == 2 || kt == 4) ? (size_t)74 * 1024
                            : p->order <= 5 ? (size_t)110 * 1024 : (size_t)220 * 1024;
      for (int psi : {64, 32}) {
        eval(psi, nullptr, lo_n, w_n, lmin_n, lmax_n);
        const int32_t wn = (dmas::bl_span(kt) + w_n + extra + 1) / 2 * 2;
        if (dmas::beamform_lds64_smem_bytes(nm, wn, p->interp, kt, psi) <= budget) {
          p->paired = 1;
          p->lds_kt = kt;
          p->lds_psi = psi;
          p->W = wn;
          qlo.swap(lo_n);
          lo_min = lmin_n;
          lo_max = lmax_n;
          break;
        }
        kd_ord = kd_order(psi);
        eval(psi, &kd_ord, lo_k, w_k, lmin_k, lmax_k);
        const int32_t wk = (dmas::bl_span(kt) + w_k + extra + 1) / 2 * 2;
        if (w_k < w_n && dmas::beamform_lds64_smem_bytes(nm, wk, p->interp, kt, psi) <= budget) {
          p->paired = 1;
          p->lds_kt = kt;
          p->lds_psi = psi;
          p->W = wk;
          qlo.swap(lo_k);
          order.swap(kd_ord);
          lo_min = lmin_k;
          lo_max = lmax_k;
          break;
        }
      }
      if (p->paired) break;
    }
  }
  const size_t smem = p->paired ? dmas::beamform_lds64_smem_bytes(nm, p->W, p->interp, p->lds_kt, p->lds_psi)
                                : dmas::beamform_smem_bytes(nm, p->W, p->interp, p->mg);
  int smem_optin = 0;
  PLAN_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem + 64 > (size_t)smem_optin)
    return bail(fail(DMAS_ERR_INVALID, "microphone count x delay spread exceeds the shared-memory window (" +
                                           std::to_string(smem) + " B)"));
  if (p->paired) {
    PLAN_TRY(dmas::beamform_lds64_configure(nm, p->W, p->interp, p->lds_kt, p->lds_psi));
    // byte offsets into the CTA's [n_mics][W] window of 8-byte columns: 8 (i W + d - lo);
    // padding microphones and directions past the grid end -> the zero block (column n_mics W)
    const size_t n_pt = qlo.size() / nm;
    const size_t n_tab = n_pt * p->lds_psi * n_pad;
    // (interpolating: the fractions alongside, padding 0)
    std::vector<int32_t> offs(n_tab, 8 * nm * p->W);
    std::vector<float> alph(p->interp ? n_tab : 0, 0.f);
    for (size_t t = 0; t < n_pt; ++t)
      for (int q = 0; q < p->lds_psi; ++q) {
        const int64_t k = (int64_t)t * p->lds_psi + q;
        if (k >= nd) break;
        const int64_t a = order.empty() ? k : order[(size_t)k];
        const size_t row = ((size_t)t * p->lds_psi + q) * n_pad;
        for (int i = 0; i < nm; ++i) {
          offs[row + i] = 8 * (i * p->W + (p->h_delays[(size_t)a * nm + i] - qlo[t * nm + i]));
          if (p->interp) alph[row + i] = p->h_alpha[(size_t)a * nm + i];
        }
      }
    // bounds audit (compute-sanitizer is unavailable on the GPU pool): a lane reads columns
    // off / 8 + lane + 64 m (+ 1 interpolating), m < kt / 2, which must stay inside the microphone's
    // own window row, or inside the zero block for padding slots
    {
      const int64_t reach = dmas::bl_span(p->lds_kt) - 1 + (p->interp ? 1 : 0);
      for (size_t e = 0; e < n_tab; ++e) {
        const int64_t col = offs[e] / 8, i = col / p->W;
        const bool pad = col == (int64_t)nm * p->W;
        if (col < 0 || (!pad && (i >= nm || col - i * p->W + reach >= p->W)) ||
            (pad && reach >= dmas::bl_zero(p->lds_kt)))
          return bail(fail(DMAS_ERR_INVALID, "internal: LDS.64 offset table leaves its window"));
      }
    }
    PLAN_TRY(cudaMalloc(&p->d_offs, n_tab * sizeof(int32_t)));
    PLAN_TRY(cudaMemcpy(p->d_offs, offs.data(), n_tab * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (p->interp) {
      PLAN_TRY(cudaMalloc(&p->d_alpha_tab, n_tab * sizeof(float)));
      PLAN_TRY(cudaMemcpy(p->d_alpha_tab, alph.data(), n_tab * sizeof(float), cudaMemcpyHostToDevice));
    }
    PLAN_TRY(cudaMalloc(&p->d_qlo, qlo.size() * sizeof(int32_t)));
    PLAN_TRY(cudaMemcpy(p->d_qlo, qlo.data(), qlo.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (!order.empty()) {
      PLAN_TRY(cudaMalloc(&p->d_psi_map, order.size() * sizeof(int32_t)));
      PLAN_TRY(cudaMemcpy(p->d_psi_map, order.data(), order.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
  } else {
    PLAN_TRY(dmas::beamform_configure(nm, p->W, p->interp, p->mg));
    PLAN_TRY(cudaMalloc(&p->d_tile_lo, tile_lo.size() * sizeof(int32_t)));
    PLAN_TRY(cudaMemcpy(p->d_tile_lo, tile_lo.data(), tile_lo.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  if (p->mg == 0 && !p->paired) {
    // classic path: every CTA of a psi tile (all t tiles, all frames) uses the same word offsets
    // i W + d - lo into its staged window (and, interpolating, the same fractions); build them once
    // here, the kernel TMA-copies its tile's [BF_PSI][n_pad] block(s) alongside the window.  Padding
    // microphones (and directions past the grid end) point at the kernel's zero block at word
    // n_mics W with fraction 0.
    const size_t n_tab = tile_lo.size() * dmas::BF_PSI * n_pad;
    std::vector<int32_t> offs(n_tab, nm * p->W);
    std::vector<float> alph(p->interp ? n_tab : 0, 0.f);
    for (size_t t = 0; t < tile_lo.size(); ++t)
      for (int q = 0; q < dmas::BF_PSI; ++q) {
        const int64_t a = (int64_t)t * dmas::BF_PSI + q;
        if (a >= nd) break;
        const size_t row = ((size_t)t * dmas::BF_PSI + q) * n_pad;
        for (int i = 0; i < nm; ++i) {
          offs[row + i] = i * p->W + (p->h_delays[(size_t)a * nm + i] - tile_lo[t]);
          if (p->interp) alph[row + i] = p->h_alpha[(size_t)a * nm + i];
        }
      }
    PLAN_TRY(cudaMalloc(&p->d_offs, n_tab * sizeof(int32_t)));
    PLAN_TRY(cudaMemcpy(p->d_offs, offs.data(), n_tab * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (p->interp) {
      PLAN_TRY(cudaMalloc(&p->d_alpha_tab, n_tab * sizeof(float)));
      PLAN_TRY(cudaMemcpy(p->d_alpha_tab, alph.data(), n_tab * sizeof(float), cudaMemcpyHostToDevice));
    }
  }

  // ---- signed-root plane with zero guards: reads at t + d outside [0, T) return 0 (reading Q5)
  // (LDS.64 path: columns of the paired plane; sample t is also stored at column G + t - 32)
  p->G = std::max<int64_t>(p->paired ? dmas::BL_STRIDE : 0, -(int64_t)lo_min);
  p->G = (p->G + 3) / 4 * 4;
  const int t_tile = p->paired ? 32 * p->lds_kt : dmas::BF_T;
  const int64_t ntt = (p->T + t_tile - 1) / t_tile;
  p->Tp = p->G + (ntt - 1) * t_tile + std::max<int64_t>(0, lo_max) + p->W;
  p->Tp = std::max<int64_t>(p->Tp, p->G + p->T);
  p->Tp = (p->Tp + 3) / 4 * 4;
  // bounds audit: every staged window [G + t0 + lo, + W) lies inside a plane row
  if (p->mg == 0 && (p->G + lo_min < 0 || p->G + (ntt - 1) * t_tile + lo_max + p->W > p->Tp))
    return bail(fail(DMAS_ERR_INVALID, "internal: staged window leaves the root plane"));
  const size_t plane_frame = (size_t)nm * p->Tp * sizeof(float) * (p->paired ? 2 : 1);
  const size_t plane_budget = (size_t)256 << 20;
  p->chunk_cap = (int32_t)std::max<size_t>(1, std::min<size_t>((size_t)p->max_frames, plane_budget / plane_frame));
  PLAN_TRY(cudaMalloc(&p->d_splane, plane_frame * p->chunk_cap));
  PLAN_TRY(cudaMemset(p->d_splane, 0, plane_frame * p->chunk_cap));

  // ---- matched filter template (zero-padded to a multiple of 4), 1 / energy in float64
  if (p->mf_taps > 0) {
    p->mf_lp = (p->mf_taps + 3) / 4 * 4;
    std::vector<float> w((size_t)p->mf_lp, 0.f);
    double e = 0.0;
    for (int k = 0; k < p->mf_taps; ++k) {
      w[k] = desc->mf_coeffs[k];
      e += (double)w[k] * w[k];
    }
    p->mf_inv_energy = (float)(1.0 / e);
    PLAN_TRY(cudaMalloc(&p->d_mf, w.size() * sizeof(float)));
    PLAN_TRY(cudaMemcpy(p->d_mf, w.data(), w.size() * sizeof(float), cudaMemcpyHostToDevice));
    PLAN_TRY(dmas::mf_configure(p->mf_lp));
  }

  // ---- envelope taps
  if (p->lp_taps > 0) {
    std::vector<double> h = blackman_lowpass(p->lp_taps, desc->lp_cutoff_hz, p->fs);
    p->h_lp.assign(h.begin(), h.end());
    PLAN_TRY(cudaMalloc(&p->d_lp, p->h_lp.size() * sizeof(float)));
    PLAN_TRY(cudaMemcpy(p->d_lp, p->h_lp.data(), p->h_lp.size() * sizeof(float), cudaMemcpyHostToDevice));
    if (p->bp_taps > 0) {
      p->h_bp.assign(desc->bp_coeffs, desc->bp_coeffs + p->bp_taps);
      PLAN_TRY(cudaMalloc(&p->d_bp, p->h_bp.size() * sizeof(float)));
      PLAN_TRY(cudaMemcpy(p->d_bp, p->h_bp.data(), p->h_bp.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    p->lp_fast = (p->lp_taps == dmas::ENV_FAST_TAPS && p->bp_taps == 0 && p->env_decim == 1 && p->T % 4 == 0);
    p->env_engine = desc->env_engine;
    p->lp_tc = (desc->env_engine != 1 && p->lp_taps <= dmas::ENV_FAST_TAPS && p->bp_taps == 0 && p->env_decim == 1 &&
                dmas::envelope_tc_supported(p->T));
    p->presplit = p->lp_tc && desc->env_engine == 0;
    if (p->lp_fast || p->lp_tc)
      for (int i = 0; i < p->lp_taps; ++i) p->lp127.h[i] = p->h_lp[i];
    if (p->lp_tc) {
      PLAN_TRY(dmas::envelope_tc_configure());
      PLAN_TRY(cudaMalloc(&p->d_tcb, dmas::envelope_tc_b_bytes()));
      PLAN_TRY(dmas::envelope_tc_prepare(p->lp127, p->lp_taps, p->d_tcb));
    }
    PLAN_TRY(cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, dev));
    // raw-image scratch for envelope-only kinds: the budget (default 4 GiB), capped at what
    // max_frames frames of all five kinds need, and never below one frame of every kind (sharded
    // plans size it with the largest shard, so the chunking is the same on every rank)
    const size_t frame_img = (size_t)(sharded ? p->n_local_max : p->n_dirs) * p->T * sizeof(float);
    const size_t all_kinds = frame_img * dmas::N_KINDS;
    size_t cap = std::min<size_t>((size_t)p->scratch_budget, all_kinds * (size_t)p->max_frames);
    cap = std::max(cap, all_kinds);
    PLAN_TRY(cudaMalloc(&p->d_scratch, cap));
    p->scratch_cap = cap;
    p->x_scratch_cap = cap;
  }
  PLAN_TRY(cudaEventCreateWithFlags(&p->ev_last, cudaEventDisableTiming));
  if (sharded) {
    // gather staging: two buffers, each at least one frame of every raw and envelope kind of the
    // largest shard (and >= 256 MiB so chunks stay long)
    const size_t frame_max = (size_t)p->n_local_max * (p->T + p->T_out) * sizeof(float) * dmas::N_KINDS;
    p->gst_cap = std::max(frame_max, (size_t)256 << 20);
    for (int b = 0; b < 2; ++b) {
      PLAN_TRY(cudaMalloc(&p->d_gst[b], p->gst_cap));
      for (cudaEvent_t* e : {&p->ev_b[b], &p->ev_c[b], &p->ev_g[b]})
        PLAN_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    PLAN_TRY(cudaEventCreateWithFlags(&p->ev_x0, cudaEventDisableTiming));
    PLAN_TRY(cudaEventCreateWithFlags(&p->ev_x1, cudaEventDisableTiming));
  }
  PLAN_TRY(cudaDeviceSynchronize());
  if (sharded) {
    // every rank built its shard: agree on the frames per exchange chunk (the minimum over ranks);
    // a rank that failed above contributed 0 from `bail`, so all ranks fail together
    int64_t v = p->chunk_cap;
    std::string err;
    p->status_exchanged = true;
    dmas_status rc = dmas::comm::allreduce_min(p->comm, &v, p->cs, err);
    if (rc != DMAS_OK) return bail(fail(rc, err));
    if (v < 1) return bail(fail(DMAS_ERR_NCCL, "another rank failed to build its plan"));
    p->x_chunk_cap = (int32_t)v;
  }
#undef PLAN_TRY
  *out = p;
  return DMAS_OK;
}

dmas_status dmas_beamform(dmas_plan_t p, const float* signals, int32_t n_frames, float* const* outs, uint32_t what,
                          void* cuda_stream) {
  if (!p) return fail(DMAS_ERR_NULL, "plan is NULL");
  if (n_frames < 0 || n_frames > p->max_frames) return fail(DMAS_ERR_SHAPE, "n_frames not in [0, max_frames]");
  uint32_t raw_k, env_k;
  dmas_status st = check_what(p, what, raw_k, env_k);
  if (st != DMAS_OK) return st;
  if (n_frames == 0) return DMAS_OK;
  if (!signals) return fail(DMAS_ERR_NULL, "signals is NULL");
  if (((uintptr_t)signals) & 3u) return fail(DMAS_ERR_SHAPE, "misaligned signals pointer");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard guard(p->device);
  return beamform_device(p, signals, n_frames, outs, raw_k, env_k, what, (cudaStream_t)cuda_stream);
}

dmas_status dmas_beamform_host(dmas_plan_t p, const float* host_signals, int32_t n_frames, float* const* host_outs,
                               uint32_t what) {
  if (!p) return fail(DMAS_ERR_NULL, "plan is NULL");
  if (n_frames < 0) return fail(DMAS_ERR_SHAPE, "n_frames < 0");
  uint32_t raw_k, env_k;
  dmas_status st = check_what(p, what, raw_k, env_k);
  if (st != DMAS_OK) return st;
  if (n_frames == 0) return DMAS_OK;
  // sharded plans: the root's host signals go in (broadcast on the device); with DMAS_GATHER the
  // images are gathered onto the root and come out into the root's host buffers (the other ranks
  // pass NULL outputs), without it every rank copies its own shard into its own host buffers
  const bool sharded = p->comm != nullptr;
  const bool gather = sharded && (what & DMAS_GATHER);
  const bool h2d = !sharded || p->rank == p->root;
  const bool d2h = !sharded || !gather || p->rank == p->root;
  const int n_out = popcount5(raw_k) + popcount5(env_k);
  if (h2d && !host_signals) return fail(DMAS_ERR_NULL, "host signals are NULL");
  if (d2h) {
    if (!host_outs) return fail(DMAS_ERR_NULL, "host outputs are NULL");
    for (int i = 0; i < n_out; ++i)
      if (!host_outs[i]) return fail(DMAS_ERR_NULL, "output pointer is NULL");
  }
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard guard(p->device);

  // frames per pipeline stage: bounded by max_frames and ~512 MiB of device output per buffer,
  // sized with quantities every rank of a sharded plan shares (whole grid when gathering, the
  // largest shard otherwise) so all ranks take the same stages; the copies move the real rows
  const int64_t rows_out = gather ? p->n_dirs_total : p->n_dirs;
  const int64_t rows_size = gather ? p->n_dirs_total : sharded ? p->n_local_max : p->n_dirs;
  std::vector<size_t> out_frame_bytes;
  size_t out_frame_total = 0;
  for (int k = 0; k < dmas::N_KINDS; ++k)
    if ((raw_k >> k) & 1u) out_frame_bytes.push_back((size_t)rows_out * p->T * sizeof(float));
  for (int k = 0; k < dmas::N_KINDS; ++k)
    if ((env_k >> k) & 1u) out_frame_bytes.push_back((size_t)rows_out * p->T_out * sizeof(float));
  for (size_t b : out_frame_bytes) out_frame_total += b;
  const size_t out_frame_size = out_frame_total / (size_t)rows_out * (size_t)rows_size;
  const bool host_io = d2h;
  const size_t sig_frame = (size_t)p->n_mics * p->T_in * sizeof(float);
  int32_t hc = (int32_t)std::max<size_t>(1, ((size_t)512 << 20) / out_frame_size);
  hc = std::min({hc, p->max_frames, n_frames});

  for (auto& s : p->hs)
    if (!s) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // (device staging: kept between calls; non-root ranks of a sharded plan hold no image staging)
  if (p->hsig_cap < sig_frame * hc || (host_io && p->hout_cap < out_frame_total * hc)) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(p->d_hsig[b]);
      cudaFree(p->d_hout[b]);
      p->d_hsig[b] = p->d_hout[b] = nullptr;
    }
    p->hsig_cap = p->hout_cap = 0;
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(cudaMalloc(&p->d_hsig[b], sig_frame * hc));
      if (host_io) CUDA_TRY(cudaMalloc(&p->d_hout[b], out_frame_total * hc));
    }
    p->hsig_cap = sig_frame * hc;
    p->hout_cap = host_io ? out_frame_total * hc : 0;
  }
  for (auto& row : p->h_ev)
    for (auto& e : row)
      if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t* h2d_done = p->h_ev[0];
  cudaEvent_t* comp_done = p->h_ev[1];
  cudaEvent_t* d2h_done = p->h_ev[2];
  dmas_status rc = DMAS_OK;
  int chunk_idx = 0;
  for (int32_t f0 = 0; f0 < n_frames && rc == DMAS_OK; f0 += hc, ++chunk_idx) {
    const int b = chunk_idx & 1;
    const int32_t nf = std::min(hc, n_frames - f0);
    if (chunk_idx >= 2) CUDA_TRY(cudaStreamWaitEvent(p->hs[0], d2h_done[b], 0));
    if (h2d)
      CUDA_TRY(cudaMemcpyAsync(p->d_hsig[b], host_signals + (size_t)f0 * p->n_mics * p->T_in, sig_frame * nf,
                               cudaMemcpyHostToDevice, p->hs[0]));
    CUDA_TRY(cudaEventRecord(h2d_done[b], p->hs[0]));
    CUDA_TRY(cudaStreamWaitEvent(p->hs[1], h2d_done[b], 0));
    if (chunk_idx >= 2) CUDA_TRY(cudaStreamWaitEvent(p->hs[1], d2h_done[b], 0));
    std::vector<float*> douts(out_frame_bytes.size());
    size_t off = 0;
    for (size_t i = 0; i < out_frame_bytes.size(); ++i) {
      douts[i] = p->d_hout[b] + off / sizeof(float);
      off += out_frame_bytes[i] * nf;
    }
    rc = beamform_device(p, p->d_hsig[b], nf, douts.data(), raw_k, env_k, gather ? DMAS_GATHER : 0u, p->hs[1]);
    if (rc != DMAS_OK) break;
    CUDA_TRY(cudaEventRecord(comp_done[b], p->hs[1]));
    CUDA_TRY(cudaStreamWaitEvent(p->hs[2], comp_done[b], 0));
    for (size_t i = 0; host_io && i < out_frame_bytes.size(); ++i)
      CUDA_TRY(cudaMemcpyAsync(host_outs[i] + (size_t)f0 * (out_frame_bytes[i] / sizeof(float)), douts[i],
                               out_frame_bytes[i] * nf, cudaMemcpyDeviceToHost, p->hs[2]));
    CUDA_TRY(cudaEventRecord(d2h_done[b], p->hs[2]));
  }
  cudaError_t e = cudaStreamSynchronize(p->hs[2]);
  cudaStreamSynchronize(p->hs[1]);
  cudaStreamSynchronize(p->hs[0]);
  if (rc != DMAS_OK) return rc;
  if (e != cudaSuccess) return fail(DMAS_ERR_CUDA, std::string("host pipeline: ") + cudaGetErrorString(e));
  return DMAS_OK;
}

dmas_status dmas_delay_table(dmas_plan_t p, int32_t* host_out) {
  if (!p || !host_out) return fail(DMAS_ERR_NULL, "NULL argument");
  std::memcpy(host_out, p->h_delays.data(), p->h_delays.size() * sizeof(int32_t));
  return DMAS_OK;
}

dmas_status dmas_delay_fraction(dmas_plan_t p, float* host_out) {
  if (!p || !host_out) return fail(DMAS_ERR_NULL, "NULL argument");
  if (!p->interp) return fail(DMAS_ERR_SHAPE, "plan uses nearest-sample delays (delay_interp == 0)");
  std::memcpy(host_out, p->h_alpha.data(), p->h_alpha.size() * sizeof(float));
  return DMAS_OK;
}

dmas_status dmas_get_plan_info(dmas_plan_t p, dmas_plan_info* info) {
  if (!p || !info) return fail(DMAS_ERR_NULL, "NULL argument");
  info->n_dirs = p->n_dirs;
  info->n_samples = p->T;
  info->n_out_samples = p->T_out;
  info->n_mics = p->n_mics;
  info->order = p->order;
  info->lp_taps = p->lp_taps;
  info->env_decim = p->env_decim;
  info->device = p->device;
  info->d_min = p->dmin;
  info->d_max = p->dmax;
  info->psi_tile = p->paired ? p->lds_psi : p->mg > 0 ? dmas::BF_PSI_MG : dmas::BF_PSI;
  info->t_tile = p->paired ? 32 * p->lds_kt : dmas::BF_T;
  info->window = p->W;
  info->chunk_frames = p->chunk_cap;
  info->bf_kernel = p->paired ? 1 : p->mg > 0 ? 2 : 0;
  info->tile_order = p->d_psi_map ? 1 : 0;
  info->n_dirs_total = p->n_dirs_total;
  info->dir_begin = p->dir0;
  info->n_ranks = p->n_ranks;
  info->rank = p->rank;
  info->root = p->root;
  info->sharded = p->comm ? 1 : 0;
  return DMAS_OK;
}

dmas_status dmas_set_timing(dmas_plan_t p, int32_t enable) {
  if (!p) return fail(DMAS_ERR_NULL, "plan is NULL");
  std::lock_guard<std::mutex> lk(p->mu);
  p->timing = enable != 0;
  return DMAS_OK;
}

dmas_status dmas_timing_read(dmas_plan_t p, double ms_out[4], int64_t count_out[4]) {
  if (!p || !ms_out || !count_out) return fail(DMAS_ERR_NULL, "NULL argument");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard guard(p->device);
  for (int k = 0; k < 4; ++k) {
    ms_out[k] = 0.0;
    count_out[k] = 0;
  }
  dmas_status rc = DMAS_OK;
  for (auto& r : p->recs) {
    cudaError_t e = cudaEventSynchronize(r.ev1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.ev0, r.ev1);
    if (e != cudaSuccess && rc == DMAS_OK) rc = fail(DMAS_ERR_CUDA, std::string("timing: ") + cudaGetErrorString(e));
    ms_out[r.kernel] += ms;
    count_out[r.kernel] += 1;
    p->ev_pool.push_back(r.ev0);
    p->ev_pool.push_back(r.ev1);
  }
  p->recs.clear();
  return rc;
}

int64_t dmas_launch_count(void) { return g_launches.load(); }

dmas_status dmas_comm_id(uint8_t id_out[DMAS_COMM_ID_BYTES]) {
  if (!id_out) return fail(DMAS_ERR_NULL, "id_out is NULL");
  std::string err;
  dmas_status rc = dmas::comm::unique_id(id_out, err);
  return rc == DMAS_OK ? rc : fail(rc, err);
}

dmas_status dmas_shard_range(int64_t n_dirs, int32_t n_ranks, int32_t rank, int64_t* g0, int64_t* g1) {
  if (!g0 || !g1) return fail(DMAS_ERR_NULL, "NULL argument");
  if (n_dirs < 0 || n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(DMAS_ERR_INVALID, "bad shard arguments");
  dmas::comm::shard_range(n_dirs, n_ranks, rank, g0, g1);
  return DMAS_OK;
}

dmas_status dmas_gather_schedule(int64_t n_dirs, int32_t n_ranks, int32_t rank, int32_t root, int32_t n_frames,
                                 int64_t row, dmas_xfer* out, int64_t cap, int64_t* n_out) {
  if (!n_out || (cap > 0 && !out)) return fail(DMAS_ERR_NULL, "NULL argument");
  if (n_dirs < 1 || n_ranks < 1 || rank < 0 || rank >= n_ranks || root < 0 || root >= n_ranks || n_frames < 0 ||
      row < 1)
    return fail(DMAS_ERR_INVALID, "bad gather-schedule arguments");
  const std::vector<dmas_xfer> xs = dmas::comm::gather_schedule(n_dirs, n_ranks, rank, root, n_frames, row);
  *n_out = (int64_t)xs.size();
  for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)xs.size()); ++i) out[i] = xs[(size_t)i];
  return DMAS_OK;
}

void dmas_destroy(dmas_plan_t p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    DeviceGuard guard(p->device);
    cudaDeviceSynchronize();
    free_plan_memory(p);
  }
  delete p;
}

const char* dmas_status_string(dmas_status s) {
  switch (s) {
    case DMAS_OK: return "DMAS_OK";
    case DMAS_ERR_NULL: return "DMAS_ERR_NULL";
    case DMAS_ERR_INVALID: return "DMAS_ERR_INVALID";
    case DMAS_ERR_ORDER: return "DMAS_ERR_ORDER";
    case DMAS_ERR_SHAPE: return "DMAS_ERR_SHAPE";
    case DMAS_ERR_CUDA: return "DMAS_ERR_CUDA";
    case DMAS_ERR_OOM: return "DMAS_ERR_OOM";
    case DMAS_ERR_NCCL: return "DMAS_ERR_NCCL";
  }
  return "DMAS_ERR_UNKNOWN";
}

const char* dmas_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
