/*
 * dmas.h — C ABI of the B200-native DMAS / CF beamforming hot path.
 *
 * Implements the beamforming stage of Jansen, Daems, Steckel, "Delay-Multiply-And-Sum
 * Beamforming for Real-Time In-Air Acoustic Imaging" (arXiv 2511.09165).  Citations are
 * PAPER.md:<line> of the paper's LaTeX source.  Problem statement: an array of
 * N microphones with signals m_i(t); a set of M directions psi; a delay look-up table
 * tau_{i,psi}; pre-steering x_i(t,psi) = m_i(t + tau_{i,psi}) (Eq. (1)); per
 * pixel (t, psi): DAS (Eq. (2)), DMAS of order p (Eqs. (5)/(6), PAPER.md:106/116,
 * evaluated through power sums and the Newton-Girard expansions PAPER.md:129-165), the
 * Coherence Factor and CF-weighted image, then envelope detection
 * (|.| then low-pass, PAPER.md:75, 5 kHz PAPER.md:253).
 *
 * Notation: this header writes n_mics for the paper's N and n_dirs for the paper's M.
 *
 * Conventions common to every call:
 *  - No C++ types, exceptions or torch types cross this boundary.  Sizes are explicit.
 *  - Every call returns a dmas_status; DMAS_OK = 0.  On error nothing the caller owns is
 *    modified except as stated, and dmas_last_error() returns a one-line message
 *    (thread-local, valid until the next call on the same thread).
 *  - Validation errors are returned synchronously, before any device work is enqueued.
 *    Asynchronous device faults surface as DMAS_ERR_CUDA at a later call or stream sync.
 *  - Device pointers must belong to the plan's device and be 4-byte aligned.
 *  - A plan is immutable after dmas_plan() (except its internal scratch, which dmas_plan
 *    allocates: a call never allocates device memory or synchronises).  Host-side, calls on
 *    one plan are serialised by an internal mutex; device-side, the work a call enqueues is
 *    ordered after the previous call's work on the same plan (a plan-owned event the new
 *    call's stream waits on), whatever streams the two calls use, because both use the
 *    plan's signed-root plane and scratch.  Distinct plans are independent.
 */
#ifndef DMAS_H
#define DMAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dmas_plan_s* dmas_plan_t;

typedef enum {
  DMAS_OK = 0,
  DMAS_ERR_NULL = 1,    /* a required pointer argument is NULL                                   */
  DMAS_ERR_INVALID = 2, /* bad descriptor value: fs<=0, c<=0, n_mics<1, n_dirs<1, n_samples<1,
                           non-finite geometry, theta not in [-pi,pi], phi not in [-pi/2,pi/2],
                           duplicate microphone positions, lp_taps even or <0, lp_cutoff not in
                           (0, fs/2), bp_taps even or <0, env_decim<1, cf_eps<0, delay range
                           too large for int32 windows                                            */
  DMAS_ERR_ORDER = 3,   /* order p not in [2,8], n_mics < p (the DMAS sum is empty), or p >= 6
                           with n_mics < 2p (fp32 Newton-Girard cancellation)     */
  DMAS_ERR_SHAPE = 4,   /* n_frames<0 or > max_frames; output mask asks for nothing / for an
                           envelope on a plan built with lp_taps == 0; misaligned pointer         */
  DMAS_ERR_CUDA = 5,    /* CUDA runtime/launch error (message in dmas_last_error())               */
  DMAS_ERR_OOM = 6,     /* device or pinned host allocation failed                                 */
  DMAS_ERR_NCCL = 7     /* sharded plans: NCCL missing, communicator setup or a collective failed  */
} dmas_status;

/* Output image kinds (bit order = order of the `outs` arrays below). */
enum {
  DMAS_KIND_DAS = 1,    /* S_DAS = sum_i x_i                              Eq. (2)   */
  DMAS_KIND_DMAS = 2,   /* S_DMAS^(p) = E_p(s_1..s_N)                     Eq. (6)  */
  DMAS_KIND_CFDMAS = 4, /* S_DMAS^(p) * CF  */
  DMAS_KIND_CFDAS = 8,  /* S_DAS * CF  ("can also be applied to DAS")  */
  DMAS_KIND_CF = 16,    /* CF = (sum x)^2 / (N sum x^2 + eps)  */
  DMAS_KIND_ALL = 31
};
/* `what` = raw-stage kinds | (envelope-stage kinds << 8) | flags. */
#define DMAS_RAW(kinds) ((uint32_t)(kinds))
#define DMAS_ENV(kinds) (((uint32_t)(kinds)) << 8)
/* Flags for direction-sharded plans (n_ranks > 1 or a comm_id; ignored by single-GPU plans):
   DMAS_GATHER: gather every requested image onto the root rank (full [F][n_dirs][.] buffers there,
   `outs` ignored on the other ranks); without it each rank's `outs` are its own shard
   [F][n_local][.] (shards stay resident).  DMAS_SIGNALS_RESIDENT: every rank already holds the
   signals, skip the broadcast from the root. */
#define DMAS_GATHER (1u << 16)
#define DMAS_SIGNALS_RESIDENT (1u << 17)
#define DMAS_COMM_ID_BYTES 128

typedef struct {
  /* Geometry (host memory, caller-owned, copied by dmas_plan). */
  int32_t n_mics;            /* N >= 1                                                          */
  const double* mic_xyz;     /* [n_mics][3] metres; x = broadside, array usually in the y-z plane */
  int64_t n_dirs;            /* M >= 1                                                          */
  const double* dir_az_el;   /* [n_dirs][2] radians (azimuth theta from +x toward +y, elevation
                                phi toward +z); row order = image row order                     */
  const double* reference_xyz; /* [3] phase centre; NULL = origin                               */
  double fs_hz;              /* sample rate, > 0                                                */
  double c_mps;              /* speed of sound, > 0                                             */
  int32_t order;             /* DMAS order p in [2,8]: 2..5 use the paper's explicit expansions
                                (PAPER.md:142-160), 6..8 the general partition formula
                                 with compile-time coefficient tables             */
  int64_t n_samples;         /* T, samples per channel per frame, >= 1                          */
  int32_t max_frames;        /* upper bound on n_frames per call, >= 1                          */
  float cf_eps;              /* CF denominator guard, >= 0; default 1e-30        */
  /* Envelope stage. */
  int32_t lp_taps;           /* odd low-pass length; 0 = plan has no envelope stage; default 127 */
  double lp_cutoff_hz;       /* (0, fs/2); default 5000; Blackman-windowed sinc, unit DC gain    */
  int32_t bp_taps;           /* optional band-pass FIR length (odd); 0 = off (default)           */
  const float* bp_coeffs;    /* [bp_taps] host, copied; applied before |.| as a centred FIR      */
  int32_t env_decim;         /* R >= 1: envelope keeps samples t = 0, R, 2R, ... (ceil(T/R))     */
  int32_t env_engine;        /* 0 = auto: tensor-core (tcgen05) low-pass with a 3-pass BF16 split
                                (error <= ~4.6e-5 of the envelope) when lp_taps <= 127, no
                                band-pass, R == 1, T % 32 == 0 and 16-byte aligned buffers,
                                else the FP32 FIR.  For envelope-only kinds the beamform then
                                writes |y| already split into BF16 hi / lo (same 4 B per pixel)
                                and the envelope reads it without a conversion pass (identical
                                values).  1 = always the FP32 FIR; 2 = the tensor-core envelope
                                on the fp32 raw image (conversion inside the envelope kernel) */
  /* Optional matched filter (pulse compression; NEXT-1).  When mf_taps > 0 the
     signals given to dmas_beamform* are RAW recordings of n_samples + mf_taps - 1 samples per
     channel, and each channel is first correlated with the emitted signal:
       m_i(t) = sum_k mf_coeffs[k] raw_i(t + k) / sum_k mf_coeffs[k]^2 ,  t in [0, n_samples)
     (an exact unit echo starting at sample t peaks at 1 at t).  0 = signals are matched-filtered. */
  int32_t mf_taps;           /* 0 (default) or 1..16384                                         */
  const float* mf_coeffs;    /* [mf_taps] host, copied (the emitted chirp)                      */
  /* Pre-steering of Eq. (1) with a fractional delay (NEXT-2): 0 = nearest sample,
     ties to even (default; the integer LUT north_star names); 1 = linear interpolation,
     x_i(t) = (1 - a) m_i(t + d) + a m_i(t + d + 1) with d = floor(v), a = v - d (SPEC's
     pre_steer); roots are then taken per pixel on the SFU instead of hoisted.                  */
  int32_t delay_interp;
  /* Runtime. */
  int32_t device;            /* CUDA device ordinal; -1 = current device                        */
  int64_t scratch_bytes;     /* budget for the plan-owned raw-image scratch used when an
                                envelope is requested without its raw image; 0 = 4 GiB.  dmas_plan
                                allocates min(budget, max_frames frames of all 5 kinds), at least
                                one frame of every kind (plans with lp_taps > 0 only)           */
  int32_t bf_engine;         /* beamform kernel: 0 = auto (the LDS.64 kernel -- paired root plane,
                                one 8-byte shared load per 2 pixels -- when delays are integer and
                                its windows fit two CTAs per SM, else the classic one); 1 = always
                                the classic kernel.  Both give bit-identical images.           */
  /* Direction sharding over GPUs, one process per GPU (north_star: "the
     direction grid is partitioned across the GPUs ...; signals are broadcast once and image tiles
     gathered with NCCL").  Every rank passes the SAME descriptor (whole array, whole grid) with
     its own `rank` and `device`; the plan keeps the contiguous slice dmas_shard_range() gives it
     and joins an NCCL communicator (created collectively inside dmas_plan: all ranks must call it).
     n_ranks == 0 and comm_id == NULL: a single-GPU plan (default).  A comm_id with n_ranks == 1 is
     a one-rank sharded plan (same images; exercises the exchange code on one GPU). */
  int32_t n_ranks;           /* ranks (processes / GPUs) sharing the grid; 0 or 1 = one          */
  int32_t rank;              /* this process's rank in [0, n_ranks)                              */
  int32_t root;              /* rank holding the signals and receiving gathered images           */
  const uint8_t* comm_id;    /* DMAS_COMM_ID_BYTES from dmas_comm_id() on one rank, shared with
                                every rank out of band (e.g. a torch.distributed broadcast).
                                An id whose first 8 bytes are "DMASLOOP" selects the in-process
                                loopback transport instead of NCCL (test infrastructure: all
                                ranks are plans of one process, driven from concurrent threads;
                                the exchange runs as event-ordered device copies with NCCL's
                                matching and completion semantics)                               */
  int32_t fused_gather;      /* sharded plans, DMAS_GATHER of envelope-only requests on the
                                tensor-core envelope: 1 = each rank's envelope kernel stores its
                                rows straight into the root's images (CUDA IPC mapping of the
                                root's buffer, TMA stores over NVLink; no staging, no send/recv),
                                followed by a stream-ordered barrier to the root; 0 = staged
                                ncclSend / ncclRecv gather (default).  Other requests always take
                                the staged gather.                                                */
} dmas_plan_desc;

/* Fill `desc` with defaults (zero geometry; order 2; cf_eps 1e-30; lp 127 taps at 5 kHz;
   bp off; env_decim 1; device -1; max_frames 1). */
void dmas_plan_desc_init(dmas_plan_desc* desc);

/* Build a plan: validates `desc`, computes the integer delay table d[psi][i] on the device
   (A1: v = ((p_i - r) . u(psi)) * (-(fs/c)) in IEEE float64 with no FMA contraction in the
   fixed order ((dx*ux + dy*uy) + dz*uz), rounded to nearest, ties to even; u(psi) from the
   host libm), the low-pass taps, and the per-tile staging metadata, and allocates the
   plan-owned signed-root scratch.  On success *out is a new plan; on error *out = NULL. */
dmas_status dmas_plan(const dmas_plan_desc* desc, dmas_plan_t* out);

/* Beamform n_frames frames, asynchronously on `cuda_stream` (a cudaStream_t; NULL = legacy
   default stream).  Returns after enqueueing.
   Sharded plans: a collective -- every rank makes the same sequence of calls with the same
   n_frames and `what`.  `signals` is a device buffer of the full shape on every rank: the root's
   holds the recording, the others' is overwritten by the root's (ncclBroadcast per frame chunk,
   overlapped with the previous chunk's compute) unless DMAS_SIGNALS_RESIDENT.  `outs` are the
   rank's shards [n_frames][n_local][.], or with DMAS_GATHER full images on the root (assembled
   by grouped ncclSend / ncclRecv of each chunk, overlapped with the next chunk's compute; NULL
   allowed on the other ranks).  Shards are bitwise the rows a single-GPU plan computes.
     signals : DEVICE, fp32 [n_frames][n_mics][n_samples] (or [.][.][n_samples + mf_taps - 1] raw
               samples when the plan has a matched filter), t contiguous, caller-owned, read-only.
     outs    : HOST array of DEVICE pointers, one per requested (stage, kind): first the raw kinds
               of `what` in bit order, then the envelope kinds in bit order.  Raw outputs are fp32
               [n_frames][n_dirs][n_samples]; envelope outputs are fp32
               [n_frames][n_dirs][ceil(n_samples / env_decim)].  Caller-owned, write-only.
     what    : DMAS_RAW(kinds) | DMAS_ENV(kinds); must request at least one output.
   Reads of m_i outside [0, n_samples) are 0.  n_frames == 0 is a no-op. */
dmas_status dmas_beamform(dmas_plan_t plan, const float* signals, int32_t n_frames,
                          float* const* outs, uint32_t what, void* cuda_stream);

/* Same computation with HOST buffers: copies the signals in, computes, copies the images out,
   pipelined in frame chunks over copy and compute streams; synchronous (returns when every
   output is in host memory).  Host buffers may be pageable, but only page-locked buffers
   (cudaHostAlloc / cudaHostRegister) overlap copies with compute.  Any n_frames >= 0 is
   accepted (not bounded by max_frames).
   Sharded plans (a collective): the root's host_signals go in (NULL elsewhere) and are broadcast
   on the device; with DMAS_GATHER in `what` the images are gathered onto the root and land in the
   root's host_outs (full [F][n_dirs][.]; NULL elsewhere); without it every rank copies its own
   shard [F][n_local][.] into its own host_outs, in parallel over the ranks' PCIe links. */
dmas_status dmas_beamform_host(dmas_plan_t plan, const float* host_signals, int32_t n_frames,
                               float* const* host_outs, uint32_t what);

/* Copy the plan's integer delay table into host memory int32 [n_dirs][n_mics] (nearest sample,
   or floor(v) when delay_interp == 1); sharded plans: the rank's own rows [n_local][n_mics]. */
dmas_status dmas_delay_table(dmas_plan_t plan, int32_t* host_out);

/* delay_interp == 1 plans only: the fractional parts a = v - floor(v) in [0, 1), fp32
   [n_dirs][n_mics]; DMAS_ERR_SHAPE for nearest-sample plans. */
dmas_status dmas_delay_fraction(dmas_plan_t plan, float* host_out);

typedef struct {
  int64_t n_dirs, n_samples, n_out_samples; /* n_out_samples = ceil(T / env_decim); n_dirs = the
                                               plan's own rows (the rank's shard when sharded) */
  int32_t n_mics, order, lp_taps, env_decim, device;
  int32_t d_min, d_max;       /* range of the delay table (samples)                          */
  int32_t psi_tile, t_tile;   /* beamform CTA tile: directions x samples                     */
  int32_t window;             /* staged columns per microphone per CTA: samples (classic kernel:
                                 t_tile + tile spread) or 8-byte sample pairs (LDS.64 kernel:
                                 t_tile - 32 + per-microphone spread)                           */
  int32_t chunk_frames;       /* frames per internal chunk                                   */
  int32_t bf_kernel;          /* beamform kernel the plan launches: 0 classic (k_beamform), 1 LDS.64
                                 (k_beamform_lds64), 2 microphone groups (k_beamform_mg)         */
  int32_t tile_order;         /* 0: CTA tiles are runs of consecutive directions; 1: compact
                                 patches from recursive bisection of the unit vectors (LDS.64
                                 path; images unaffected)                                        */
  int64_t n_dirs_total;       /* the whole grid (== n_dirs unless sharded)                       */
  int64_t dir_begin;          /* first grid row of this plan's shard (0 unless sharded)          */
  int32_t n_ranks, rank, root;/* 1, 0, 0 unless sharded                                          */
  int32_t sharded;            /* 1: the plan holds an NCCL communicator                          */
} dmas_plan_info;
dmas_status dmas_get_plan_info(dmas_plan_t plan, dmas_plan_info* info);

/* Per-kernel device timing: when enabled, the plan records a CUDA event pair around every
   kernel it launches (on the launching stream).  dmas_timing_read synchronises those events,
   writes the summed milliseconds and launch counts per kernel (index 0 delay_table,
   1 prologue (signed roots), 2 beamform, 3 envelope) and clears the record. */
dmas_status dmas_set_timing(dmas_plan_t plan, int32_t enable);
dmas_status dmas_timing_read(dmas_plan_t plan, double ms_out[4], int64_t count_out[4]);

/* ---- Multi-GPU helpers (host only; no device work) */

/* A fresh NCCL unique id for dmas_plan_desc.comm_id (call on ONE rank, share the bytes).
   DMAS_ERR_NCCL when libnccl.so.2 cannot be loaded. */
dmas_status dmas_comm_id(uint8_t id_out[DMAS_COMM_ID_BYTES]);

/* The contiguous slice [*g0, *g1) of n_dirs grid rows that `rank` of `n_ranks` owns: sizes differ
   by at most one, the first n_dirs % n_ranks ranks hold one more. */
dmas_status dmas_shard_range(int64_t n_dirs, int32_t n_ranks, int32_t rank, int64_t* g0, int64_t* g1);

/* One point-to-point transfer of a gather (see dmas_gather_schedule). */
enum { DMAS_XFER_SEND = 0, DMAS_XFER_RECV = 1, DMAS_XFER_COPY = 2 };
typedef struct {
  int32_t kind;      /* DMAS_XFER_*                                                              */
  int32_t peer;      /* the other rank (the root for SEND; the sender for RECV; self for COPY)   */
  int32_t frame;     /* frame within the chunk                                                   */
  int32_t reserved;
  int64_t src_elem;  /* SEND / COPY: float offset into the rank's shard [n_frames][n_local][row]  */
  int64_t dst_elem;  /* RECV / COPY: float offset into the root's image [n_frames][n_dirs][row]   */
  int64_t count;     /* floats                                                                    */
} dmas_xfer;

/* The exact list of transfers `rank` performs when a sharded plan gathers one image of an
   n_frames chunk (row = floats per image row) onto `root`, in issue order: per frame, per rank,
   the root RECVs (or COPYs its own) rows [g0_r, g1_r) and each other rank SENDs its rows.  The
   library executes this list (COPYs as device copies, the rest in one ncclGroupStart/End);
   exposed so the exchange can be checked without GPUs.  Writes at most `cap` entries to `out`
   (may be NULL when cap == 0) and the full count to *n_out. */
dmas_status dmas_gather_schedule(int64_t n_dirs, int32_t n_ranks, int32_t rank, int32_t root, int32_t n_frames,
                                 int64_t row, dmas_xfer* out, int64_t cap, int64_t* n_out);

/* Total number of kernels this library has launched in the process (all plans). */
int64_t dmas_launch_count(void);

/* Destroy a plan (NULL-safe).  Synchronises the plan's device work first. */
void dmas_destroy(dmas_plan_t plan);

const char* dmas_status_string(dmas_status status);
const char* dmas_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* DMAS_H */
