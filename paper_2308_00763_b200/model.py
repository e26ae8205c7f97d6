"""State-space model, template and synthetic-video input (drop-in for halfpf.model).

Mirrors /root/reference/pkg/src/halfpf/model.py's public data types and the
input side of the tracking step:

  ModelParams      model.py:27-49   (same fields, defaults and validation)
  PixelTemplate    model.py:52-66
  disk_template    model.py:69-78   (same offset order: dy outer, dx inner)
  Video            model.py:81-102
  generate_video   model.py:123-157 (same NumPy PCG64 stream -> same bytes)
  PFVD container   model.py:270-297, truth CSV 300-316

Video synthesis is host NumPy on purpose: it is the input generator, not the
tracking step (OUT OF SCOPE row; "next" row 8f-2).  The
likelihood itself is evaluated only on the device (csrc/pf_kernels.cuh).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class ModelParams:
    drift_x: float = 1.0
    std_x: float = 5.0
    drift_y: float = 2.0
    std_y: float = 2.0
    bg_mean: float = 100.0
    fg_mean: float = 228.0
    likelihood_scale: float = 50.0
    disk_radius: int = 5
    noise_std: float = 5.0

    def __post_init__(self):
        if self.std_x <= 0 or self.std_y <= 0:
            raise ValueError("transition standard deviations must be positive")
        if self.noise_std < 0:
            raise ValueError("noise_std must be non-negative")
        if self.bg_mean == self.fg_mean:
            raise ValueError("background and foreground means must differ")
        if self.disk_radius < 1:
            raise ValueError("disk_radius must be at least 1")


@dataclass(frozen=True)
class PixelTemplate:
    offsets: np.ndarray  # (N, 2) int64, columns (dx, dy)

    def __post_init__(self):
        o = np.asarray(self.offsets, dtype=np.int64)
        if o.ndim != 2 or o.shape[1] != 2:
            raise ValueError("offsets must have shape (N, 2)")
        object.__setattr__(self, "offsets", o)

    @property
    def count(self) -> int:
        return int(self.offsets.shape[0])


def disk_template(radius: int) -> PixelTemplate:
    r = int(radius)
    span = np.arange(-r, r + 1)
    dy, dx = np.meshgrid(span, span, indexing="ij")  # row-major: dy outer, dx inner
    keep = dx * dx + dy * dy <= r * r
    return PixelTemplate(np.stack([dx[keep], dy[keep]], axis=1).astype(np.int64))


@dataclass
class Video:
    frames: np.ndarray  # (F, H, W) uint8
    truth: np.ndarray  # (F, 2) float64 (x, y)

    def __post_init__(self):
        if len(self.frames) != len(self.truth):
            raise ValueError("truth length must match frame count")

    @property
    def frame_count(self) -> int:
        return int(self.frames.shape[0])

    @property
    def height(self) -> int:
        return int(self.frames.shape[1])

    @property
    def width(self) -> int:
        return int(self.frames.shape[2])


def _bounce(pos: float, step: float, hi: float) -> Tuple[float, float]:
    """Specular reflection off [0, hi] (model.py:105-120)."""
    pos += step
    while pos < 0.0 or pos > hi:
        if pos < 0.0:
            pos, step = -pos, -step
        if pos > hi:
            pos, step = 2.0 * hi - pos, -step
    return pos, step


def _check_bounce(params: ModelParams, width: int, height: int) -> None:
    # the reference's bounce loop (model.py:105-121) never ends on a 1-pixel
    # axis with a non-zero drift; refuse instead of hanging
    if (width == 1 and params.drift_x != 0.0) or (height == 1 and params.drift_y != 0.0):
        raise ValueError("a 1-pixel frame axis with non-zero drift has no bounded trajectory")


def generate_video(params: ModelParams, frames: int, width: int, height: int,
                   start: Tuple[float, float], seed: int) -> Video:
    if frames < 1:
        raise ValueError("frames must be at least 1")
    _check_bounce(params, width, height)
    x, y = float(start[0]), float(start[1])
    if not (0.0 <= x <= width - 1 and 0.0 <= y <= height - 1):
        raise ValueError(f"start {start} outside frame bounds {width}x{height}")
    gen = np.random.Generator(np.random.PCG64(seed))
    offs = disk_template(params.disk_radius).offsets
    vx, vy = params.drift_x, params.drift_y
    truth = np.empty((frames, 2), dtype=np.float64)
    out = np.empty((frames, height, width), dtype=np.uint8)
    for t in range(frames):
        truth[t] = (x, y)
        canvas = np.full((height, width), params.bg_mean, dtype=np.float64)
        cx, cy = int(round(x)), int(round(y))
        canvas[np.clip(offs[:, 1] + cy, 0, height - 1), np.clip(offs[:, 0] + cx, 0, width - 1)] = params.fg_mean
        if params.noise_std > 0:
            canvas += gen.normal(0.0, params.noise_std, size=canvas.shape)
        out[t] = np.clip(np.rint(canvas), 0, 255).astype(np.uint8)
        x, vx = _bounce(x, vx, width - 1.0)
        y, vy = _bounce(y, vy, height - 1.0)
    return Video(frames=out, truth=truth)


_MAGIC = b"PFVD"


def write_video(path, video: Video) -> None:
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<III", video.frame_count, video.width, video.height))
        fh.write(np.ascontiguousarray(video.frames, dtype=np.uint8).tobytes())


def read_video(path) -> np.ndarray:
    with open(path, "rb") as fh:
        if fh.read(4) != _MAGIC:
            raise ValueError(f"{path}: bad container magic at offset 0")
        hdr = fh.read(12)
        if len(hdr) != 12:
            raise ValueError(f"{path}: truncated header at offset 4")
        n, w, h = struct.unpack("<III", hdr)
        body = fh.read()
    if len(body) != n * w * h:
        raise ValueError(f"{path}: expected {n * w * h} pixel bytes at offset 16, got {len(body)}")
    return np.frombuffer(body, dtype=np.uint8).reshape(n, h, w).copy()


def write_truth_csv(path, truth: np.ndarray) -> None:
    with open(path, "w", newline="") as fh:
        fh.write("frame,x,y\n")
        for t, (x, y) in enumerate(np.asarray(truth, dtype=np.float64)):
            fh.write(f"{t},{float(x)!r},{float(y)!r}\n")


def read_truth_csv(path) -> np.ndarray:
    with open(path) as fh:
        head = fh.readline().strip()
        if head != "frame,x,y":
            raise ValueError(f"{path}: unexpected truth CSV header {head!r}")
        rows = [tuple(float(v) for v in line.strip().split(",")[1:]) for line in fh if line.strip()]
    return np.array(rows, dtype=np.float64).reshape(-1, 2)


# --- device-side input ----------------------------------------


def _lib():
    from . import _native

    return _native


def generate_video_device(params: ModelParams, frames: int, width: int, height: int,
                          start: Tuple[float, float], seed: int, device: int = 0):
    """The reference video model rendered on the device (pf_generate_video).

    Returns (frames: torch uint8 CUDA tensor [F, H, W], truth: (F, 2) float64).
    Same model and trajectory as generate_video; the pixel noise comes from the
    counter-based LCG stream of `seed` instead of NumPy's PCG64 (frames are a
    pure function of (seed, t, y, x); oracle/video.py restates them)."""
    import ctypes as C

    import torch

    N = _lib()
    if frames < 1:
        raise ValueError("frames must be at least 1")
    _check_bounce(params, width, height)
    x, y = float(start[0]), float(start[1])
    if not (0.0 <= x <= width - 1 and 0.0 <= y <= height - 1):
        raise ValueError(f"start {start} outside frame bounds {width}x{height}")
    out = torch.empty((frames, height, width), dtype=torch.uint8, device=torch.device("cuda", device))
    truth = np.empty((frames, 2), dtype=np.float64)
    offs = np.ascontiguousarray(disk_template(params.disk_radius).offsets.astype(np.int32))
    p = N.pf_params(params.drift_x, params.std_x, params.drift_y, params.std_y, params.bg_mean, params.fg_mean,
                    params.likelihood_scale, params.disk_radius, params.noise_std)
    rc = N.lib().pf_generate_video(C.byref(p), int(frames), int(width), int(height), x, y,
                                   int(seed) & ((1 << 64) - 1), N.ptr(offs), int(offs.shape[0]),
                                   C.c_void_p(out.data_ptr()), N.ptr(truth), int(device))
    N.check(rc, N.lib().pf_global_error)
    return out, truth


def read_video_device(path, device: int = 0):
    """PFVD container -> torch uint8 CUDA tensor [F, H, W] (pinned, double-buffered ingest)."""
    import ctypes as C

    import torch

    N = _lib()
    fwh = np.zeros(3, dtype=np.int32)
    bpath = str(path).encode()
    rc = N.lib().pf_pfvd_info(bpath, N.ptr(fwh))
    if rc == N.PF_EIO:
        msg = N.lib().pf_global_error().decode()
        if msg.endswith("cannot open"):
            raise FileNotFoundError(msg)
        raise ValueError(msg)
    N.check(rc, N.lib().pf_global_error)
    F, W, H = (int(v) for v in fwh)
    out = torch.empty((F, H, W), dtype=torch.uint8, device=torch.device("cuda", device))
    rc = N.lib().pf_read_pfvd(bpath, C.c_void_p(out.data_ptr()), out.numel(), N.ptr(fwh), int(device))
    if rc == N.PF_EIO:
        raise ValueError(N.lib().pf_global_error().decode())
    N.check(rc, N.lib().pf_global_error)
    return out
