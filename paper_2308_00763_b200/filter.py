"""Drop-in tracking API over the sm_100a kernels (mirrors halfpf.filter).

Reference interface (/root/reference/pkg/src/halfpf/filter.py) -> here:

  PrecisionMode / from_name   :49-60   same values and error message
  DegeneracyError(frame)      :63-68   same type, .frame set by run()
  RngStream                   :71-82   same methods; the product stream is the
                                       counter-based LCG,
                                       generated on the device
  ParticleSet                 :85-134  device-resident; *_f64(), snapshot(),
                                       settable fields (stage_hook edits)
  _validate_k / MAX_PARTICLES :137-143 same messages; the 65536 bound of the
                                       CPU emulation is lifted to 2^31-1 per
                                       track
  RunResult                   :146-151 same fields (op counters are zero:
                                       out of scope, ncu replaces them)
  make_engine + stage methods :154-567 staged engine, one device call per
                                       reference stage (reference semantics,
                                       incl. the sequential binary16 folds)
  init_particles              :573-580
  systematic_ancestors        :583-588 device kernel
  run                         :591-662 fused one-launch-per-frame path;
                                       with stage_hook -> staged engine

New: `Filter` -- per-frame step / batched independent tracks on one device.
"""

from __future__ import annotations

import ctypes as C
import enum
import math
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .model import ModelParams, PixelTemplate, Video, disk_template

MAX_PARTICLES = (1 << 31) - 1
STAGES = ("propagate", "likelihood", "max", "weight", "normalize", "resample")


class PrecisionMode(enum.Enum):
    FP64 = "fp64"
    FP32 = "fp32"
    FP16_SCALAR = "fp16"
    FP16_PACKED = "fp16-packed"

    @classmethod
    def from_name(cls, name: str) -> "PrecisionMode":
        for m in cls:
            if m.value == name:
                return m
        raise ValueError(f"unknown precision {name!r}")


_NATIVE_MODE = {
    PrecisionMode.FP64: N.PF_FP64,
    PrecisionMode.FP32: N.PF_FP32,
    PrecisionMode.FP16_SCALAR: N.PF_FP16,
    PrecisionMode.FP16_PACKED: N.PF_FP16_PACKED,
}
_DTYPE = {
    PrecisionMode.FP64: np.float64,
    PrecisionMode.FP32: np.float32,
    PrecisionMode.FP16_SCALAR: np.float16,
    PrecisionMode.FP16_PACKED: np.float16,
}


def _mode(mode) -> PrecisionMode:
    return mode if isinstance(mode, PrecisionMode) else PrecisionMode.from_name(str(mode))


class DegeneracyError(RuntimeError):
    """All particle weights collapsed to zero (or went non-finite)."""

    def __init__(self, message: str, frame: Optional[int] = None):
        super().__init__(message)
        self.frame = frame


@dataclass
class OpCounters:
    """Reference op counters (halfnum.py:40-67).  Out of scope on the GPU
    (SURVEY.md 2): kept for API compatibility, always zero; ncu pipe metrics
    are the B200 evidence instead."""

    widen_count: int = 0
    narrow_count: int = 0
    half_arith_count: int = 0
    wide_arith_count: int = 0
    special_fn_count: int = 0

    @property
    def conversion_count(self) -> int:
        return self.widen_count + self.narrow_count


@dataclass
class RunResult:
    trajectory: np.ndarray
    counters: OpCounters
    stage_ms: Dict[str, float]
    total_ms: float
    launches: int = 0
    timings_ms: Dict[str, float] = field(default_factory=dict)


def _validate_k(K: int, mode: PrecisionMode) -> None:
    if K < 2:
        raise ValueError("particle count must be at least 2")
    if K > MAX_PARTICLES:
        raise ValueError(f"particle count {K} exceeds the {MAX_PARTICLES} bound")
    if mode is PrecisionMode.FP16_PACKED and K % 2:
        raise ValueError("packed binary16 mode requires an even particle count")


def _params_struct(p: ModelParams) -> N.pf_params:
    return N.pf_params(p.drift_x, p.std_x, p.drift_y, p.std_y, p.bg_mean, p.fg_mean,
                       p.likelihood_scale, int(p.disk_radius), p.noise_std)


def _offsets(template: PixelTemplate) -> np.ndarray:
    return np.ascontiguousarray(template.offsets.astype(np.int32).reshape(-1))


# ---------------------------------------------------------------------------
# RNG stream (device-generated LCG draws)
# ---------------------------------------------------------------------------


class RngStream:
    """Counter-based LCG stream with the reference's RngStream interface.

    `normals(K)` consumes 2K stream positions (C order: x then y per
    particle), `uniform()` one -- the order the fused kernel assumes, so a
    staged run that draws from this stream reproduces the fused run's draws.
    """

    def __init__(self, seed: int, device: int = 0):
        self.seed = int(seed) & ((1 << 64) - 1)
        self.device = device
        self.pos = 0

    def normals(self, n: int) -> np.ndarray:
        out = np.empty(2 * n, dtype=np.float64)
        N.check(N.lib().pf_rng_normals(self.seed, self.pos, 2 * n, N.ptr(out), self.device),
                N.lib().pf_global_error)
        self.pos += 2 * n
        return out.reshape(n, 2)

    def uniform(self) -> float:
        out = np.empty(1, dtype=np.float64)
        N.check(N.lib().pf_rng_uniforms(self.seed, self.pos, 1, N.ptr(out), self.device),
                N.lib().pf_global_error)
        self.pos += 1
        return float(out[0])


class PhiloxRngStream:
    """The reference's own stream, Generator(Philox(seed)) (filter.py:71-82),
    generated on the device (NumPy's Philox4x64-10 counter/buffer semantics,
    NumPy's ziggurat, glibc's log1p).  Inject it as `filter.RngStream` to run
    the staged engine on exactly the reference's draws.  The Philox key comes
    from NumPy's SeedSequence expansion of the seed (host seeding only)."""

    def __init__(self, seed: int, device: int = 0):
        st = np.random.Philox(seed).state
        state = np.array(list(st["state"]["key"]) + list(st["state"]["counter"]) + list(st["buffer"]) +
                         [st["buffer_pos"]], dtype=np.uint64)
        h = C.c_void_p()
        N.check(N.lib().pf_philox_create(C.byref(h), N.ptr(state), device), N.lib().pf_global_error)
        self._h = h
        self.seed = seed

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                N.lib().pf_philox_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def normals(self, n: int) -> np.ndarray:
        out = np.empty(2 * n, dtype=np.float64)
        N.check(N.lib().pf_philox_normals(self._h, 2 * n, N.ptr(out)), N.lib().pf_global_error)
        return out.reshape(n, 2)

    def uniform(self) -> float:
        out = np.empty(1, dtype=np.float64)
        N.check(N.lib().pf_philox_uniforms(self._h, 1, N.ptr(out)), N.lib().pf_global_error)
        return float(out[0])


# ---------------------------------------------------------------------------
# staged engine (reference semantics)
# ---------------------------------------------------------------------------

_FIELDS = {"xs": 0, "ys": 1, "loglik": 2, "weights": 3, "cdf": 4, "ancestors": 5}


class ParticleSet:
    """Device-resident structure of arrays (filter.py:85-134).

    Field reads copy device -> host (NumPy array in the mode dtype, float16
    for the binary16 modes; ancestors int64).  Assigning a field uploads it
    (arrays in any float dtype are cast; for binary16 modes a list of 16-bit
    patterns, as the reference stores them, is accepted too)."""

    def __init__(self, engine: "StagedEngine", mode: PrecisionMode, count: int):
        object.__setattr__(self, "_engine", engine)
        object.__setattr__(self, "mode", mode)
        object.__setattr__(self, "count", count)

    def _get(self, name: str) -> np.ndarray:
        e = self._engine
        if name == "ancestors":
            out = np.empty(self.count, dtype=np.int64)
        else:
            out = np.empty(self.count, dtype=_DTYPE[self.mode])
        N.check(N.lib().pf_stage_get(e._h, _FIELDS[name], N.ptr(out)), e._err)
        return out

    def _set(self, name: str, value) -> None:
        e = self._engine
        if name == "ancestors":
            arr = np.ascontiguousarray(np.asarray(value, dtype=np.int64))
        else:
            dt = _DTYPE[self.mode]
            if dt is np.float16 and isinstance(value, (list, tuple)) and value and isinstance(value[0], (int, np.integer)):
                arr = np.ascontiguousarray(np.asarray(value, dtype=np.uint16).view(np.float16))
            else:
                with np.errstate(over="ignore"):
                    arr = np.ascontiguousarray(np.asarray(value, dtype=np.float64).astype(dt))
        if arr.shape != (self.count,):
            raise ValueError(f"{name} must have shape ({self.count},)")
        N.check(N.lib().pf_stage_set(e._h, _FIELDS[name], N.ptr(arr)), e._err)

    def __getattr__(self, name):
        if name in _FIELDS:
            return self._get(name)
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in _FIELDS:
            self._set(name, value)
        else:
            object.__setattr__(self, name, value)

    def _f64(self, name):
        return self._get(name).astype(np.float64)

    def xs_f64(self):
        return self._f64("xs")

    def ys_f64(self):
        return self._f64("ys")

    def loglik_f64(self):
        return self._f64("loglik")

    def weights_f64(self):
        return self._f64("weights")

    def cdf_f64(self):
        return self._f64("cdf")

    def snapshot(self) -> dict:
        return {k: self._get(k) for k in _FIELDS}


class StagedEngine:
    """One device call per reference stage (filter.py:172-567)."""

    def __init__(self, mode, params: Optional[ModelParams] = None, template: Optional[PixelTemplate] = None,
                 counters: Optional[OpCounters] = None, workers: int = 1, device: int = 0):
        self.mode = _mode(mode)
        self.params = params or ModelParams()
        self.template = template if template is not None else disk_template(self.params.disk_radius)
        self.counters = counters if counters is not None else OpCounters()
        self.workers = max(1, int(workers))
        self.device = device
        self._h = None

    def _err(self):
        return N.lib().pf_stage_error(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                N.lib().pf_stage_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def init(self, K: int, start_hint: Tuple[float, float]) -> ParticleSet:
        _validate_k(K, self.mode)
        L = N.lib()
        if self._h:
            L.pf_stage_destroy(self._h)
            self._h = None
        h = C.c_void_p()
        offs = _offsets(self.template)
        ps_ = _params_struct(self.params)
        N.check(L.pf_stage_create(C.byref(h), _NATIVE_MODE[self.mode], K, C.byref(ps_), N.ptr(offs),
                                  self.template.count, self.device), L.pf_global_error)
        self._h = h
        N.check(L.pf_stage_init(h, float(start_hint[0]), float(start_hint[1])), self._err)
        return ParticleSet(self, self.mode, K)

    def propagate(self, ps: ParticleSet, noise: np.ndarray) -> None:
        noise = np.ascontiguousarray(np.asarray(noise, dtype=np.float64).reshape(ps.count, 2))
        N.check(N.lib().pf_stage_propagate(self._h, N.ptr(noise)), self._err)

    def likelihoods(self, ps: ParticleSet, frame: np.ndarray) -> None:
        f = np.ascontiguousarray(np.asarray(frame, dtype=np.uint8))
        h, w = f.shape
        N.check(N.lib().pf_stage_likelihood(self._h, N.ptr(f), w, h), self._err)

    def max_loglik(self, ps: ParticleSet):
        m = C.c_double()
        N.check(N.lib().pf_stage_max(self._h, C.byref(m)), self._err)
        return _DTYPE[self.mode](m.value)

    def weight_update(self, ps: ParticleSet, m) -> float:
        tot = C.c_double()
        rc = N.lib().pf_stage_weight(self._h, float(m), C.byref(tot))
        if rc == N.PF_EDEGENERATE:
            raise DegeneracyError(f"weight sum degenerated to {tot.value}")
        N.check(rc, self._err)
        if self.mode in (PrecisionMode.FP16_SCALAR, PrecisionMode.FP16_PACKED):
            return float(tot.value)
        return _DTYPE[self.mode](tot.value)

    def normalize_and_scan(self, ps: ParticleSet, total) -> None:
        N.check(N.lib().pf_stage_normalize(self._h, float(total)), self._err)

    def estimate(self, ps: ParticleSet) -> Tuple[float, float]:
        ex, ey = C.c_double(), C.c_double()
        N.check(N.lib().pf_stage_estimate(self._h, C.byref(ex), C.byref(ey)), self._err)
        return float(ex.value), float(ey.value)

    def resample(self, ps: ParticleSet, u: float) -> None:
        N.check(N.lib().pf_stage_resample(self._h, float(u)), self._err)


def make_engine(mode, params: Optional[ModelParams] = None, template: Optional[PixelTemplate] = None,
                counters: Optional[OpCounters] = None, workers: int = 1, device: int = 0) -> StagedEngine:
    return StagedEngine(mode, params, template, counters, workers, device)


def init_particles(K: int, start_hint, mode, params: Optional[ModelParams] = None,
                   counters: Optional[OpCounters] = None) -> ParticleSet:
    return make_engine(mode, params, counters=counters).init(K, start_hint)


def systematic_ancestors(cdf: np.ndarray, u: float, device: int = 0) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(cdf, dtype=np.float64))
    out = np.empty(len(c), dtype=np.int64)
    N.check(N.lib().pf_systematic_ancestors(N.ptr(c), len(c), float(u), N.ptr(out), device),
            N.lib().pf_global_error)
    return out


# ---------------------------------------------------------------------------
# fused path
# ---------------------------------------------------------------------------


def _current_stream(device: int) -> int:
    """torch's current CUDA stream on `device` (raw cudaStream_t)."""
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # one call, no Stream object
    if raw is not None:
        return int(raw(device))
    return torch.cuda.current_stream(device).cuda_stream


class Filter:
    """Fused one-launch-per-frame filter on one device.

    n_tracks independent filters (seeds[i], video i % n_videos) share every
    launch -- the batched-track configuration.  `step(frame)` runs one frame
    and returns the estimate(s); `run(frames)` a whole video.
    """

    def __init__(self, K: int, mode="fp16", width: int = 128, height: int = 128, seed: int = 42,
                 params: Optional[ModelParams] = None, template: Optional[PixelTemplate] = None,
                 start_hint: Optional[Tuple[float, float]] = None, n_tracks: int = 1,
                 seeds: Optional[Sequence[int]] = None, n_videos: int = 1, tpb: Optional[int] = None,
                 device: int = 0, rng: str = "lcg"):
        if rng not in ("lcg", "numpy-philox"):
            raise ValueError(f"unknown rng {rng!r} (expected 'lcg' or 'numpy-philox')")
        self.rng = rng
        self.mode = _mode(mode)
        _validate_k(K, self.mode)
        self.K = int(K)
        self.width, self.height = int(width), int(height)
        self.params = params or ModelParams()
        self.template = template if template is not None else disk_template(self.params.disk_radius)
        self.n_tracks = int(n_tracks)
        self.n_videos = int(n_videos)
        if seeds is None:
            seeds = [int(seed) + i for i in range(self.n_tracks)]
        if len(seeds) != self.n_tracks:
            raise ValueError("need one seed per track")
        self.seeds = np.ascontiguousarray(np.asarray([int(s) & ((1 << 64) - 1) for s in seeds], dtype=np.uint64))
        if start_hint is None:
            start_hint = (self.width / 2.0, self.height / 2.0)
        self.start_hint = (float(start_hint[0]), float(start_hint[1]))
        self._offs = _offsets(self.template)
        cfg = N.pf_config()
        cfg.precision = _NATIVE_MODE[self.mode]
        cfg.K = self.K
        cfg.width, cfg.height = self.width, self.height
        cfg.n_tracks, cfg.n_videos = self.n_tracks, self.n_videos
        cfg.seeds = self.seeds.ctypes.data_as(C.POINTER(C.c_uint64))
        cfg.params = _params_struct(self.params)
        cfg.offsets_xy = self._offs.ctypes.data_as(C.POINTER(C.c_int32))
        cfg.n_offsets = self.template.count
        cfg.tpb = int(tpb or 0)
        cfg.device = int(device)
        cfg.start_x, cfg.start_y = self.start_hint
        L = N.lib()
        h = C.c_void_p()
        rc = L.pf_create(C.byref(h), C.byref(cfg))
        if rc == N.PF_EINVAL:
            raise ValueError(L.pf_global_error().decode())
        N.check(rc, L.pf_global_error)
        self._h = h
        self.device = device
        if rng == "numpy-philox":
            # the reference's stream (filter.py:71-82): NumPy seeds the Philox
            # key (SeedSequence) on the host, the draws are generated on the device
            st = np.random.Philox(int(self.seeds[0])).state
            state = np.array(list(st["state"]["key"]) + list(st["state"]["counter"]) + list(st["buffer"]) +
                             [st["buffer_pos"]], dtype=np.uint64)
            rc = L.pf_set_rng_philox(h, N.ptr(state))
            if rc:
                msg = self._err().decode()
                self.close()
                raise ValueError(msg)

    def _err(self):
        return N.lib().pf_last_error(self._h)

    def close(self):
        if getattr(self, "_h", None):
            N.lib().pf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, start_hint: Optional[Tuple[float, float]] = None):
        if start_hint is not None:
            self.start_hint = (float(start_hint[0]), float(start_hint[1]))
        N.check(N.lib().pf_reset(self._h, *self.start_hint), self._err)

    def _frames_arg(self, frames, n_frames: Optional[int]):
        """Validate frames against the handle and return (pointer, on_device, keepalive, n_frames).

        Accepted: [n_videos][F][H][W] uint8, or [F][H][W] with one video
        (n_frames=None); for one frame ([n_videos][H][W] / [H][W]) pass
        n_frames=1 with the frame axis absent.  Host arrays must be uint8
        (C-contiguous copies are made as needed); CUDA tensors must be uint8,
        contiguous and on the handle's device (they are read in place)."""
        H, W, nv = self.height, self.width, self.n_videos
        is_cuda = hasattr(frames, "data_ptr") and getattr(frames, "is_cuda", False)
        shape = tuple(int(v) for v in frames.shape)
        if n_frames == 1 and len(shape) in (2, 3) and shape[-2:] == (H, W) and (len(shape) == 2 or shape[0] == nv):
            shape = (nv, 1, H, W) if len(shape) == 3 else (1, H, W)
        if len(shape) == 3 and nv == 1:
            shape = (1,) + shape
        if len(shape) != 4 or shape[0] != nv or shape[2:] != (H, W) or shape[1] < 1:
            want = f"({nv}, F, {H}, {W})" + (f" or (F, {H}, {W})" if nv == 1 else "")
            raise ValueError(f"frames of shape {tuple(frames.shape)} do not match the filter: expected {want}")
        F = shape[1]
        if n_frames is not None and n_frames != F:
            raise ValueError(f"expected {n_frames} frame(s), got {F}")
        if is_cuda:
            import torch

            if frames.dtype != torch.uint8:
                raise ValueError(f"frames must be uint8, got {frames.dtype}")
            if not frames.is_contiguous():
                raise ValueError("CUDA frames must be contiguous")
            if frames.device.index != self.device:
                raise ValueError(f"CUDA frames are on device {frames.device.index}, the filter on {self.device}")
            return C.c_void_p(frames.data_ptr()), 1, frames, F
        arr = np.asarray(frames)
        if arr.dtype != np.uint8:
            raise ValueError(f"frames must be uint8, got {arr.dtype}")
        arr = np.ascontiguousarray(arr)
        return C.c_void_p(arr.ctypes.data), 0, arr, F

    def _launch(self, frames, n_frames: Optional[int]) -> np.ndarray:
        p, on_dev, keep, F = self._frames_arg(frames, n_frames)
        traj = np.empty((self.n_tracks, F, 2), dtype=np.float64)
        L = N.lib()
        if on_dev:
            # device frames may still be in flight on torch's current stream:
            # the library stream is ordered after it (no host synchronisation),
            # then the synchronous call (one-frame steps: zero-copy result)
            rc = L.pf_stream_wait(self._h, C.c_void_p(_current_stream(self.device)))
            if rc == N.PF_OK:
                rc = L.pf_run(self._h, p, F, 1, N.ptr(traj))
        else:
            rc = L.pf_run(self._h, p, F, 0, N.ptr(traj))
        del keep
        if rc == N.PF_EDEGENERATE:
            raise DegeneracyError(self._err().decode(), L.pf_degenerate_frame(self._h))
        N.check(rc, self._err)
        return traj

    def run_frames(self, frames, n_frames: Optional[int] = None) -> np.ndarray:
        """frames: [n_videos][F][H][W] (or [F][H][W] with one video) -> [n_tracks][F][2]."""
        return self._launch(frames, n_frames)

    def run(self, frames) -> np.ndarray:
        traj = self._launch(frames, None)
        return traj[0] if self.n_tracks == 1 else traj

    def step(self, frame):
        """One frame ([H][W], or [n_videos][H][W]) -> the estimate(s) (filter.py:617-654)."""
        est = self._launch(frame, 1)[:, 0, :]
        return (float(est[0, 0]), float(est[0, 1])) if self.n_tracks == 1 else est

    def run_async(self, frames, traj_out, stream=None):
        """Stream-ordered run of CUDA frames into a CUDA float64 tensor traj_out
        [n_tracks][F][2]: queued behind `stream` (default: torch's current
        stream), which later work can consume without a host synchronisation.
        Call sync() to wait and to surface a DegeneracyError."""
        import torch

        p, on_dev, keep, F = self._frames_arg(frames, None)
        if not on_dev:
            raise ValueError("run_async takes CUDA frames")
        if (not getattr(traj_out, "is_cuda", False) or traj_out.dtype != torch.float64 or not traj_out.is_contiguous()
                or tuple(traj_out.shape) != (self.n_tracks, F, 2)):
            raise ValueError(f"traj_out must be a contiguous CUDA float64 tensor of shape ({self.n_tracks}, {F}, 2)")
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._async_keep = (keep, traj_out)
        N.check(N.lib().pf_run_async(self._h, p, F, 1, C.c_void_p(traj_out.data_ptr()), C.c_void_p(s)), self._err)

    def sync(self):
        rc = N.lib().pf_sync(self._h)
        self._async_keep = None
        if rc == N.PF_EDEGENERATE:
            raise DegeneracyError(self._err().decode(), N.lib().pf_degenerate_frame(self._h))
        N.check(rc, self._err)

    def likelihood_maps(self, frames) -> np.ndarray:
        """[F, H+2r, W+2r] per-position likelihood maps of host frames (mode dtype)."""
        arr = np.ascontiguousarray(np.asarray(frames, dtype=np.uint8))
        if arr.ndim == 2:
            arr = arr[None]
        r = int(np.max(np.abs(self._offs))) if self._offs.size else 0
        out = np.empty((arr.shape[0], self.height + 2 * r, self.width + 2 * r), dtype=_DTYPE[self.mode])
        N.check(N.lib().pf_likelihood_maps(self._h, N.ptr(arr), int(arr.shape[0]), N.ptr(out)), self._err)
        return out

    def timings(self) -> Dict[str, float]:
        t = (C.c_float * 6)()
        N.check(N.lib().pf_last_timings(self._h, t), self._err)
        keys = ("total", "upload", "maps", "frames", "tables", "download")
        return {k: float(v) for k, v in zip(keys, t)}

    def set_profiling(self, on: bool = True):
        N.check(N.lib().pf_set_profiling(self._h, int(bool(on))), self._err)

    def launches(self) -> int:
        return int(N.lib().pf_last_launches(self._h))

    def state(self, track: int = 0):
        dt = _DTYPE[self.mode]
        xs = np.empty(self.K, dtype=dt)
        ys = np.empty(self.K, dtype=dt)
        cdf = np.empty(self.K, dtype=dt)
        N.check(N.lib().pf_get_state(self._h, track, N.ptr(xs), N.ptr(ys), N.ptr(cdf)), self._err)
        return xs, ys, cdf

    def set_state(self, xs, ys, frame: int, track: int = 0):
        """Inject post-resample positions entering frame `frame` (teacher forcing):
        the next frame uses identity ancestors and frame `frame`'s draws
        (pf_set_state; the reference's seam is a stage_hook editing ParticleSet)."""
        dt = _DTYPE[self.mode]
        with np.errstate(over="ignore"):
            x = np.ascontiguousarray(np.asarray(xs).astype(dt, copy=False))
            y = np.ascontiguousarray(np.asarray(ys).astype(dt, copy=False))
        if x.shape != (self.K,) or y.shape != (self.K,):
            raise ValueError(f"xs and ys must have shape ({self.K},)")
        N.check(N.lib().pf_set_state(self._h, int(track), N.ptr(x), N.ptr(y), int(frame)), self._err)

    def enable_debug(self):
        N.check(N.lib().pf_get_debug(self._h, 0, None, None), self._err)

    def debug(self, track: int = 0):
        anc = np.empty(self.K, dtype=np.int64)
        L = np.empty(self.K, dtype=_DTYPE[self.mode])
        N.check(N.lib().pf_get_debug(self._h, track, N.ptr(anc), N.ptr(L)), self._err)
        return anc, L


def run(video: Video, K: int, mode, seed: int, workers: int = 1, params: Optional[ModelParams] = None,
        template: Optional[PixelTemplate] = None, start_hint: Optional[Tuple[float, float]] = None,
        stage_hook: Optional[Callable] = None, tpb: Optional[int] = None, device: int = 0,
        engine: Optional[str] = None, rng: str = "lcg") -> RunResult:
    """Track through a whole video (filter.py:591-662).

    engine="fused" (default without stage_hook): one fused kernel + one tile
    table kernel per frame, FP16 is the stabilised variant.  engine="staged"
    (forced by stage_hook): one device call per reference stage, reference
    semantics in every mode, draws from `RngStream` (resolved at call time,
    so it can be swapped, as in the reference).  rng="numpy-philox" draws
    from the reference's own stream, Generator(Philox(seed)), on the device
    (both engines)."""
    mode = _mode(mode)
    params = params or ModelParams()
    template = template if template is not None else disk_template(params.disk_radius)
    _validate_k(K, mode)
    if start_hint is None:
        start_hint = (video.width / 2.0, video.height / 2.0)
    if engine is None:
        engine = "staged" if stage_hook is not None else "fused"
    if engine == "fused":
        if stage_hook is not None:
            raise ValueError("stage_hook requires engine='staged'")
        f = Filter(K, mode, video.width, video.height, seed, params, template, start_hint, tpb=tpb, device=device,
                   rng=rng)
        try:
            t0 = time.perf_counter()
            try:
                traj = f.run(video.frames)
            except DegeneracyError:
                raise
            wall = (time.perf_counter() - t0) * 1e3
            tm = f.timings()
            stage_ms = {name: 0.0 for name in STAGES}
            stage_ms["likelihood"] = tm["maps"]
            stage_ms["propagate"] = tm["frames"]
            return RunResult(trajectory=traj, counters=OpCounters(), stage_ms=stage_ms, total_ms=max(wall, tm["total"]),
                             launches=f.launches(), timings_ms=tm)
        finally:
            f.close()
    if engine != "staged":
        raise ValueError(f"unknown engine {engine!r}")
    eng = make_engine(mode, params, template, device=device)
    if rng not in ("lcg", "numpy-philox"):
        raise ValueError(f"unknown rng {rng!r} (expected 'lcg' or 'numpy-philox')")
    stream = PhiloxRngStream(seed, device) if rng == "numpy-philox" else RngStream(seed)
    ps = eng.init(K, start_hint)
    trajectory = np.empty((video.frame_count, 2), dtype=np.float64)
    stage_ms = {name: 0.0 for name in STAGES}
    t_start = time.perf_counter()
    for t in range(video.frame_count):
        frame = video.frames[t]
        try:
            t0 = time.perf_counter()
            eng.propagate(ps, stream.normals(K))
            t1 = time.perf_counter()
            if stage_hook:
                stage_hook(t, "propagate", ps)
            eng.likelihoods(ps, frame)
            t2 = time.perf_counter()
            if stage_hook:
                stage_hook(t, "likelihood", ps)
            m = eng.max_loglik(ps)
            t3 = time.perf_counter()
            if stage_hook:
                stage_hook(t, "max", ps)
            total = eng.weight_update(ps, m)
            t4 = time.perf_counter()
            if stage_hook:
                stage_hook(t, "weight", ps)
            eng.normalize_and_scan(ps, total)
            trajectory[t] = eng.estimate(ps)
            t5 = time.perf_counter()
            if stage_hook:
                stage_hook(t, "normalize", ps)
            eng.resample(ps, stream.uniform())
            t6 = time.perf_counter()
            if stage_hook:
                stage_hook(t, "resample", ps)
        except DegeneracyError as err:
            err.frame = t
            raise
        for name, a, b in zip(STAGES, (t0, t1, t2, t3, t4, t5), (t1, t2, t3, t4, t5, t6)):
            stage_ms[name] += (b - a) * 1e3
    total_ms = (time.perf_counter() - t_start) * 1e3
    return RunResult(trajectory=trajectory, counters=OpCounters(), stage_ms=stage_ms, total_ms=total_ms)


def accuracy_metrics(trajectory: np.ndarray, truth: np.ndarray) -> Tuple[float, float, float]:
    """(rmse, mean, max) Euclidean error (bench.py:46-61)."""
    a = np.asarray(trajectory, dtype=np.float64)
    b = np.asarray(truth, dtype=np.float64)
    if len(a) != len(b):
        raise ValueError(f"trajectory length {len(a)} != truth length {len(b)}")
    e = np.hypot(a[:, 0] - b[:, 0], a[:, 1] - b[:, 1])
    return float(np.sqrt(np.mean(e ** 2))), float(np.mean(e)), float(np.max(e))
