"""Thin ctypes binding of include/dmas.h (argument marshalling only).

Every step of the beamforming path runs in libdmas.so's sm_100a kernels; this module only
packs descriptors, passes device pointers (torch tensors' ``data_ptr()``) and the current
CUDA stream, and turns status codes into exceptions.  There is no CPU fallback: if the
shared library is missing or fails to load, importing this module raises.
"""

from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("DMAS_LIBRARY") or os.path.join(_PKG, "libdmas.so")   # override: experiments only

KIND_DAS, KIND_DMAS, KIND_CFDMAS, KIND_CFDAS, KIND_CF = 1, 2, 4, 8, 16
KIND_ALL = 31
KIND_BITS = {"das": KIND_DAS, "dmas": KIND_DMAS, "cfdmas": KIND_CFDMAS, "cfdas": KIND_CFDAS, "cf": KIND_CF}
KIND_ORDER = ("das", "dmas", "cfdmas", "cfdas", "cf")     # bit order = order of `outs`

STATUS = {0: "DMAS_OK", 1: "DMAS_ERR_NULL", 2: "DMAS_ERR_INVALID", 3: "DMAS_ERR_ORDER", 4: "DMAS_ERR_SHAPE",
          5: "DMAS_ERR_CUDA", 6: "DMAS_ERR_OOM", 7: "DMAS_ERR_NCCL"}
GATHER = 1 << 16             # sharded plans: gather the images onto the root
SIGNALS_RESIDENT = 1 << 17   # sharded plans: every rank already holds the signals (no broadcast)
COMM_ID_BYTES = 128
XFER_SEND, XFER_RECV, XFER_COPY = 0, 1, 2


def RAW(kinds: int) -> int:
    return int(kinds) & KIND_ALL


def ENV(kinds: int) -> int:
    return (int(kinds) & KIND_ALL) << 8


class DmasError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


class dmas_plan_desc(ctypes.Structure):
    _fields_ = [
        ("n_mics", ctypes.c_int32),
        ("mic_xyz", ctypes.POINTER(ctypes.c_double)),
        ("n_dirs", ctypes.c_int64),
        ("dir_az_el", ctypes.POINTER(ctypes.c_double)),
        ("reference_xyz", ctypes.POINTER(ctypes.c_double)),
        ("fs_hz", ctypes.c_double),
        ("c_mps", ctypes.c_double),
        ("order", ctypes.c_int32),
        ("n_samples", ctypes.c_int64),
        ("max_frames", ctypes.c_int32),
        ("cf_eps", ctypes.c_float),
        ("lp_taps", ctypes.c_int32),
        ("lp_cutoff_hz", ctypes.c_double),
        ("bp_taps", ctypes.c_int32),
        ("bp_coeffs", ctypes.POINTER(ctypes.c_float)),
        ("env_decim", ctypes.c_int32),
        ("env_engine", ctypes.c_int32),
        ("mf_taps", ctypes.c_int32),
        ("mf_coeffs", ctypes.POINTER(ctypes.c_float)),
        ("delay_interp", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("scratch_bytes", ctypes.c_int64),
        ("bf_engine", ctypes.c_int32),
        ("n_ranks", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("root", ctypes.c_int32),
        ("comm_id", ctypes.POINTER(ctypes.c_uint8)),
        ("fused_gather", ctypes.c_int32),
    ]


class dmas_plan_info(ctypes.Structure):
    _fields_ = [
        ("n_dirs", ctypes.c_int64), ("n_samples", ctypes.c_int64), ("n_out_samples", ctypes.c_int64),
        ("n_mics", ctypes.c_int32), ("order", ctypes.c_int32), ("lp_taps", ctypes.c_int32),
        ("env_decim", ctypes.c_int32), ("device", ctypes.c_int32), ("d_min", ctypes.c_int32),
        ("d_max", ctypes.c_int32), ("psi_tile", ctypes.c_int32), ("t_tile", ctypes.c_int32),
        ("window", ctypes.c_int32), ("chunk_frames", ctypes.c_int32), ("bf_kernel", ctypes.c_int32),
        ("tile_order", ctypes.c_int32), ("n_dirs_total", ctypes.c_int64), ("dir_begin", ctypes.c_int64),
        ("n_ranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("root", ctypes.c_int32), ("sharded", ctypes.c_int32),
    ]


class dmas_xfer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("peer", ctypes.c_int32), ("frame", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("src_elem", ctypes.c_int64), ("dst_elem", ctypes.c_int64),
                ("count", ctypes.c_int64)]


# The exported C symbols (include/dmas.h).  tests/test_abi.py checks the .so exports each.
EXPORTS = ("dmas_plan_desc_init", "dmas_plan", "dmas_beamform", "dmas_beamform_host", "dmas_delay_table",
           "dmas_delay_fraction",
           "dmas_get_plan_info", "dmas_set_timing", "dmas_timing_read", "dmas_launch_count", "dmas_destroy",
           "dmas_status_string", "dmas_last_error", "dmas_comm_id", "dmas_shard_range", "dmas_gather_schedule")


def _load() -> ctypes.CDLL:
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    lib.dmas_plan_desc_init.argtypes = [ctypes.POINTER(dmas_plan_desc)]
    lib.dmas_plan_desc_init.restype = None
    lib.dmas_plan.argtypes = [ctypes.POINTER(dmas_plan_desc), ctypes.POINTER(P)]
    lib.dmas_plan.restype = ctypes.c_int
    lib.dmas_beamform.argtypes = [P, P, ctypes.c_int32, ctypes.POINTER(P), ctypes.c_uint32, P]
    lib.dmas_beamform.restype = ctypes.c_int
    lib.dmas_beamform_host.argtypes = [P, P, ctypes.c_int32, ctypes.POINTER(P), ctypes.c_uint32]
    lib.dmas_beamform_host.restype = ctypes.c_int
    lib.dmas_delay_table.argtypes = [P, P]
    lib.dmas_delay_table.restype = ctypes.c_int
    lib.dmas_delay_fraction.argtypes = [P, P]
    lib.dmas_delay_fraction.restype = ctypes.c_int
    lib.dmas_get_plan_info.argtypes = [P, ctypes.POINTER(dmas_plan_info)]
    lib.dmas_get_plan_info.restype = ctypes.c_int
    lib.dmas_set_timing.argtypes = [P, ctypes.c_int32]
    lib.dmas_set_timing.restype = ctypes.c_int
    lib.dmas_timing_read.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    lib.dmas_timing_read.restype = ctypes.c_int
    lib.dmas_launch_count.argtypes = []
    lib.dmas_launch_count.restype = ctypes.c_int64
    lib.dmas_destroy.argtypes = [P]
    lib.dmas_destroy.restype = None
    lib.dmas_status_string.argtypes = [ctypes.c_int]
    lib.dmas_status_string.restype = ctypes.c_char_p
    lib.dmas_last_error.argtypes = []
    lib.dmas_last_error.restype = ctypes.c_char_p
    lib.dmas_comm_id.argtypes = [P]
    lib.dmas_comm_id.restype = ctypes.c_int
    lib.dmas_shard_range.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int64)]
    lib.dmas_shard_range.restype = ctypes.c_int
    lib.dmas_gather_schedule.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int64, P, ctypes.c_int64,
                                         ctypes.POINTER(ctypes.c_int64)]
    lib.dmas_gather_schedule.restype = ctypes.c_int
    return lib


lib = _load()


def _check(status: int):
    if status != 0:
        raise DmasError(status, lib.dmas_last_error().decode(errors="replace"))


def launch_count() -> int:
    return int(lib.dmas_launch_count())


def comm_id() -> bytes:
    """dmas_comm_id: a fresh NCCL unique id (call on one rank, share the bytes with the others)."""
    buf = (ctypes.c_uint8 * COMM_ID_BYTES)()
    _check(lib.dmas_comm_id(buf))
    return bytes(buf)


def loopback_comm_id() -> bytes:
    """A comm id for the library's in-process loopback transport (include/dmas.h comm_id): the
    ranks of a sharded plan as plans of this process driven from concurrent threads (tests)."""
    return b"DMASLOOP" + os.urandom(COMM_ID_BYTES - 8)


def shard_range(n_dirs: int, n_ranks: int, rank: int):
    """dmas_shard_range: the contiguous grid rows [g0, g1) `rank` owns."""
    g0, g1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.dmas_shard_range(int(n_dirs), int(n_ranks), int(rank), ctypes.byref(g0), ctypes.byref(g1)))
    return int(g0.value), int(g1.value)


def gather_schedule(n_dirs: int, n_ranks: int, rank: int, root: int, n_frames: int, row: int):
    """dmas_gather_schedule: the transfers `rank` performs to gather one image of an n_frames chunk
    onto `root`, as a list of dicts (kind, peer, frame, src_elem, dst_elem, count)."""
    n = ctypes.c_int64()
    _check(lib.dmas_gather_schedule(n_dirs, n_ranks, rank, root, n_frames, row, None, 0, ctypes.byref(n)))
    arr = (dmas_xfer * max(1, n.value))()
    _check(lib.dmas_gather_schedule(n_dirs, n_ranks, rank, root, n_frames, row, arr, n.value, ctypes.byref(n)))
    return [{f: getattr(arr[i], f) for f, _ in dmas_xfer._fields_ if f != "reserved"} for i in range(n.value)]


def _f64(a, shape_last):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2 or a.shape[1] != shape_last:
        raise ValueError(f"expected [n][{shape_last}] array, got {a.shape}")
    return a


def _current_stream_ptr(device: int):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Plan:
    """Owns a ``dmas_plan_t``.  Names and arguments follow include/dmas.h."""

    def __init__(self, mic_xyz, dir_az_el, fs: float, c: float, order: int, n_samples: int, *,
                 max_frames: int = 1, reference_xyz=None, cf_eps: float = 1e-30, lp_taps: int = 127,
                 lp_cutoff_hz: float = 5000.0, bp_coeffs: Optional[Sequence[float]] = None, env_decim: int = 1,
                 device: int = -1, scratch_bytes: int = 0, env_engine: int = 0,
                 mf_coeffs: Optional[Sequence[float]] = None, delay_interp: int = 0, bf_engine: int = 0,
                 n_ranks: int = 0, rank: int = 0, root: int = 0, comm_id: Optional[bytes] = None,
                 fused_gather: int = 0):
        self._h = ctypes.c_void_p()
        self._keep = []
        mic = _f64(mic_xyz, 3)
        dirs = _f64(dir_az_el, 2)
        d = dmas_plan_desc()
        lib.dmas_plan_desc_init(ctypes.byref(d))
        d.n_mics = mic.shape[0]
        d.mic_xyz = mic.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        d.n_dirs = dirs.shape[0]
        d.dir_az_el = dirs.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        if reference_xyz is not None:
            ref = np.ascontiguousarray(np.asarray(reference_xyz, dtype=np.float64).reshape(3))
            self._keep.append(ref)
            d.reference_xyz = ref.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        d.fs_hz, d.c_mps, d.order, d.n_samples = float(fs), float(c), int(order), int(n_samples)
        d.max_frames, d.cf_eps, d.lp_taps, d.lp_cutoff_hz = int(max_frames), float(cf_eps), int(lp_taps), float(lp_cutoff_hz)
        if bp_coeffs is not None and len(bp_coeffs) > 0:
            bp = np.ascontiguousarray(np.asarray(bp_coeffs, dtype=np.float32))
            self._keep.append(bp)
            d.bp_taps = bp.shape[0]
            d.bp_coeffs = bp.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        d.env_decim, d.device, d.scratch_bytes = int(env_decim), int(device), int(scratch_bytes)
        d.env_engine = int(env_engine)
        d.delay_interp = int(delay_interp)
        d.bf_engine = int(bf_engine)
        self.mf_taps = 0
        if mf_coeffs is not None and len(mf_coeffs) > 0:
            mf = np.ascontiguousarray(np.asarray(mf_coeffs, dtype=np.float32))
            self._keep.append(mf)
            d.mf_taps = self.mf_taps = mf.shape[0]
            d.mf_coeffs = mf.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        if comm_id is not None:
            if len(comm_id) != COMM_ID_BYTES:
                raise ValueError(f"comm_id must be {COMM_ID_BYTES} bytes")
            cid = (ctypes.c_uint8 * COMM_ID_BYTES).from_buffer_copy(comm_id)
            self._keep.append(cid)
            d.comm_id = ctypes.cast(cid, ctypes.POINTER(ctypes.c_uint8))
        d.n_ranks, d.rank, d.root = int(n_ranks), int(rank), int(root)
        d.fused_gather = int(fused_gather)
        self._keep += [mic, dirs]
        _check(lib.dmas_plan(ctypes.byref(d), ctypes.byref(self._h)))
        info = dmas_plan_info()
        _check(lib.dmas_get_plan_info(self._h, ctypes.byref(info)))
        self.info = {name: getattr(info, name) for name, _ in dmas_plan_info._fields_}
        self.n_mics, self.n_dirs = int(info.n_mics), int(info.n_dirs)
        self.n_samples, self.n_out_samples = int(info.n_samples), int(info.n_out_samples)
        self.order, self.max_frames = int(info.order), int(max_frames)
        self.device = int(info.device)
        self.n_dirs_total, self.dir_begin = int(info.n_dirs_total), int(info.dir_begin)
        self.sharded, self.rank, self.root = bool(info.sharded), int(info.rank), int(info.root)

    # -- dmas_delay_table
    def delay_table(self) -> np.ndarray:
        out = np.empty((self.n_dirs, self.n_mics), dtype=np.int32)
        _check(lib.dmas_delay_table(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    # -- dmas_delay_fraction (linear pre-steering plans)
    def delay_fraction(self) -> np.ndarray:
        out = np.empty((self.n_dirs, self.n_mics), dtype=np.float32)
        _check(lib.dmas_delay_fraction(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def out_shapes(self, n_frames: int, what: int):
        """(stage, kind, shape) of each output in `outs` order; a sharded plan's shards are
        [F][n_local][.], gathered images (what & GATHER) [F][n_dirs_total][.] on the root."""
        raw_k, env_k = what & KIND_ALL, (what >> 8) & KIND_ALL
        rows = self.n_dirs_total if (self.sharded and what & GATHER) else self.n_dirs
        shapes = []
        for name in KIND_ORDER:
            if raw_k & KIND_BITS[name]:
                shapes.append(("raw", name, (n_frames, rows, self.n_samples)))
        for name in KIND_ORDER:
            if env_k & KIND_BITS[name]:
                shapes.append(("env", name, (n_frames, rows, self.n_out_samples)))
        return shapes

    # -- dmas_beamform (device buffers, async on the current torch stream)
    def beamform(self, signals, what: int, outs: Optional[list] = None, stream=None) -> Dict:
        import torch
        if not (isinstance(signals, torch.Tensor) and signals.is_cuda and signals.dtype == torch.float32):
            raise TypeError("signals must be a CUDA float32 tensor [F][n_mics][T]")
        n_in = self.n_samples + max(0, self.mf_taps - 1)
        if not signals.is_contiguous() or signals.dim() != 3 or signals.shape[1:] != (self.n_mics, n_in):
            raise ValueError(f"signals must be contiguous [F][{self.n_mics}][{n_in}], got {tuple(signals.shape)}")
        if signals.device.index != self.device:
            raise ValueError(f"signals are on cuda:{signals.device.index}, the plan on cuda:{self.device}")
        F = signals.shape[0]
        shapes = self.out_shapes(F, what)
        if self.sharded and what & GATHER and self.rank != self.root:
            # gathered onto the root: this rank computes its shard into plan staging and sends it
            st = ctypes.c_void_p(stream) if isinstance(stream, int) else (
                ctypes.c_void_p(stream.cuda_stream) if stream is not None else _current_stream_ptr(self.device))
            _check(lib.dmas_beamform(self._h, ctypes.c_void_p(signals.data_ptr()), F, None, what, st))
            return {}
        if outs is None:
            outs = [torch.empty(s, dtype=torch.float32, device=signals.device) for (_, _, s) in shapes]
        if len(outs) != len(shapes):
            raise ValueError(f"{len(outs)} output buffers for {len(shapes)} requested outputs")
        for o, (_, _, s) in zip(outs, shapes):
            if tuple(o.shape) != s or o.dtype != torch.float32 or not o.is_contiguous() or not o.is_cuda:
                raise ValueError(f"output buffer must be contiguous float32 {s}")
            if o.device.index != self.device:
                raise ValueError(f"output buffer on cuda:{o.device.index}, the plan on cuda:{self.device}")
        arr = (ctypes.c_void_p * max(1, len(outs)))(*[o.data_ptr() for o in outs])
        st = ctypes.c_void_p(stream) if isinstance(stream, int) else (
            ctypes.c_void_p(stream.cuda_stream) if stream is not None else _current_stream_ptr(self.device))
        _check(lib.dmas_beamform(self._h, ctypes.c_void_p(signals.data_ptr()), F, arr, what, st))
        return {(stage, name): o for (stage, name, _), o in zip(shapes, outs)}

    # -- dmas_beamform_host (host buffers, synchronous, pipelined copies)
    def beamform_host(self, signals: Optional[np.ndarray], what: int, outs: Optional[list] = None,
                      n_frames: Optional[int] = None) -> Dict:
        """Host buffers in and out (synchronous).  Sharded plans: a collective; the root passes the
        recording (the other ranks pass signals=None and n_frames); with GATHER in `what` the root
        receives the whole images and the other ranks get {}, without it every rank receives its
        own shard [F][n_local][.] in host memory."""
        if self.sharded and self.rank != self.root:
            F = int(n_frames)
            if what & GATHER:
                _check(lib.dmas_beamform_host(self._h, None, F, None, what))
                return {}
            shapes = self.out_shapes(F, what)
            if outs is None:
                outs = [np.empty(s, dtype=np.float32) for (_, _, s) in shapes]
            if len(outs) != len(shapes):
                raise ValueError(f"{len(outs)} output buffers for {len(shapes)} requested outputs")
            for o, (_, _, s) in zip(outs, shapes):
                if o.shape != s or o.dtype != np.float32 or not o.flags.c_contiguous:
                    raise ValueError(f"output buffer must be contiguous float32 {s}")
            arr = (ctypes.c_void_p * max(1, len(outs)))(*[_host_ptr(o) for o in outs])
            _check(lib.dmas_beamform_host(self._h, None, F, arr, what))
            return {(stage, name): o for (stage, name, _), o in zip(shapes, outs)}
        if signals.dtype != np.float32 or not signals.flags.c_contiguous:
            raise TypeError("signals must be C-contiguous float32")
        if signals.ndim != 3 or signals.shape[1:] != (self.n_mics, self.n_samples + max(0, self.mf_taps - 1)):
            raise ValueError("signals must be [F][n_mics][T (+ mf_taps - 1)]")
        F = signals.shape[0]
        shapes = self.out_shapes(F, what)
        if outs is None:
            outs = [np.empty(s, dtype=np.float32) for (_, _, s) in shapes]
        if len(outs) != len(shapes):
            raise ValueError(f"{len(outs)} output buffers for {len(shapes)} requested outputs")
        for o, (_, _, s) in zip(outs, shapes):
            if o.shape != s or o.dtype != np.float32 or not o.flags.c_contiguous:
                raise ValueError(f"output buffer must be contiguous float32 {s}")
        arr = (ctypes.c_void_p * max(1, len(outs)))(*[_host_ptr(o) for o in outs])
        _check(lib.dmas_beamform_host(self._h, ctypes.c_void_p(_host_ptr(signals)), F, arr, what))
        return {(stage, name): o for (stage, name, _), o in zip(shapes, outs)}

    # -- per-kernel device timing
    def set_timing(self, enable: bool):
        _check(lib.dmas_set_timing(self._h, 1 if enable else 0))

    def timing_read(self):
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        _check(lib.dmas_timing_read(self._h, ms, cnt))
        names = ("delay_table", "signed_roots", "beamform", "envelope")
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(names)}

    def close(self):
        if self._h:
            lib.dmas_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _host_ptr(a) -> int:
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()      # pinned torch CPU tensor


# C-ABI names (same names as include/dmas.h)
def dmas_plan(*args, **kw) -> Plan:
    return Plan(*args, **kw)


def dmas_beamform(plan: Plan, signals, what: int, outs=None, stream=None):
    return plan.beamform(signals, what, outs, stream)


def dmas_beamform_host(plan: Plan, signals, what: int, outs=None):
    return plan.beamform_host(signals, what, outs)


def dmas_delay_table(plan: Plan):
    return plan.delay_table()


def dmas_destroy(plan: Plan):
    plan.close()
