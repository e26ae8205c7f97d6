"""ORACLE (test infrastructure only) -- the device video renderer restated
(csrc/pf_video.cuh, pf_generate_video).

Reference model: model.generate_video (/root/reference/pkg/src/halfpf/
model.py:123-157): background, disk template stamped at the half-even-rounded
centre with clipped offsets, `img += normal(0, std)` (base + std*z), rint, clip
to [0, 255]; truth by the specular-bounce recurrence (:105-121).  The only
change: z for pixel (t, y, x) is the LCG ziggurat normal at position
(t*H + y)*W + x of the video stream (oracle/rng.py).
"""

from __future__ import annotations

import numpy as np

from . import rng
from .reference_port import Params, disk_offsets


def video_stream_state(seed: int) -> int:
    return rng.splitmix64_mix(rng.lcg_seed_state(seed) ^ 0x56494445)


def _bounce(pos, step, hi):
    pos += step
    while pos < 0.0 or pos > hi:
        if pos < 0.0:
            pos, step = -pos, -step
        if pos > hi:
            pos, step = 2.0 * hi - pos, -step
    return pos, step


def generate_video_lcg(params: Params, frames: int, width: int, height: int, start, seed: int):
    offs = disk_offsets(params.disk_radius)
    x, y = float(start[0]), float(start[1])
    vx, vy = params.drift_x, params.drift_y
    truth = np.empty((frames, 2), dtype=np.float64)
    n = frames * height * width
    z = rng.normals_from_lcg_words(rng.lcg_words(video_stream_state(seed), 0, n)).reshape(frames, height, width)
    out = np.empty((frames, height, width), dtype=np.uint8)
    for t in range(frames):
        truth[t] = (x, y)
        canvas = np.full((height, width), params.bg_mean, dtype=np.float64)
        cx, cy = int(round(x)), int(round(y))
        canvas[np.clip(offs[:, 1] + cy, 0, height - 1), np.clip(offs[:, 0] + cx, 0, width - 1)] = params.fg_mean
        if params.noise_std > 0:
            canvas = canvas + params.noise_std * z[t]
        out[t] = np.clip(np.rint(canvas), 0, 255).astype(np.uint8)
        x, vx = _bounce(x, vx, width - 1.0)
        y, vy = _bounce(y, vy, height - 1.0)
    return out, truth
