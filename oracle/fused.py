"""ORACLE (test infrastructure only) -- restatement of the fused tile algorithm.

This is the CPU statement of the product's one-pass-per-frame algorithm
(DESIGN.md "Fused frame algorithm"); the CUDA path must match it BIT-EXACTLY
in all three precisions.  It is in turn compared with the reference-semantics
oracle (oracle/reference_port.py), which restates halfpf's `run()`
(/root/reference/pkg/src/halfpf/filter.py:591-662):

  * FP64 / FP32: same draws (oracle.rng LCG stream), same propagation
    arithmetic (filter.py:195-202: (x[a]+d(drift)) + d(std)*d(n), no FMA),
    same likelihood (filter.py:204-217, via the bit-identical per-position
    map), same systematic points (filter.py:248-255: (d(k)+d(u))/d(K)).  The
    weight sum / CDF are computed hierarchically in exact fixed point (tile-
    local max shift, integer scans), so they differ from NumPy's float
    cumsum by rounding only; trajectories agree to 1e-9 (FP64) / 1e-4 (FP32).
  * FP16: the north star's stabilised variant.  Propagation (filter.py:346-382),
    likelihood (filter.py:384-423) and exp16 (halfnum.py:254-263) are the
    reference's binary16 semantics; the max shift is tile-local, the weights
    w16 = exp16(RN16(L - m_tile)) are summed exactly as integers (w16*2^20),
    and the CDF is stored rescaled per tile (c = RN16(cum/S_tile)), so it
    never saturates at large K (the reference's fp16 cumsum stalls).

Per-frame structure (T = TILE particles per tile, n tiles, track = one filter):
  1. ancestors: t == 0 -> identity; else source tile b = last b with s_b <= k,
     local coordinate q = clamp((p_k - O_b) * invM_b, 0, 1) with the mode's
     systematic point p_k (FP64/FP32: the reference formulas), or for FP16 the
     f32 tile-local q = ((k - s_b) + phi_b) * rho_b, phi_b = f32(s_b + u - K O_b),
     rho_b = f32(1/(K M_b)); a_k = b*T + lower_bound(c_tile_b, q).
  2. propagate with the LCG normals of (t, k); likelihood = map lookup.
  3. tile: m_b = max L; w_q = rint(exp(L - m_b) * 2^F); cum = inclusive scan;
     S_b = sum; c_j = d(cum_j / S_b) (forced 1 where cum_j == S_b);
     X_b, Y_b = position moments (int64 for FP16, canonical pairwise f64 tree
     for FP32/FP64).
  4. tile table: m = max m_b; f_b = exp64(m_b - m); mass_q = rint(S_b*f_b*2^(Q-F));
     exact int64 prefix -> O_b, invM_b; s_b = #points <= O_b; estimate =
     tree(f_b*X_b) / tree(f_b*S_b).
"""

from __future__ import annotations

import math
from typing import Optional, Tuple

import numpy as np

from . import rng
from .reference_port import (
    F16,
    Params,
    disk_offsets,
    exp16_table,
    loglik_map_half,
    loglik_map_wide,
    lookup,
)

TILE = 1024
FBITS = {"fp64": 52, "fp32": 40, "fp16": 20}
XQ_BITS = 10  # FP16 position quantum for the estimate moments
DT = {"fp64": np.float64, "fp32": np.float32, "fp16": np.float16}


def qbits(n_tiles: int) -> int:
    return 52 - int(math.ceil(math.log2(max(1, n_tiles))))


def pairwise_tree(v: np.ndarray, axis_len_pow2: int) -> np.ndarray:
    """Canonical pairwise tree sum over the last axis (length padded to pow2)."""
    v = np.asarray(v, dtype=np.float64)
    n = v.shape[-1]
    if n < axis_len_pow2:
        pad = np.zeros(v.shape[:-1] + (axis_len_pow2 - n,), dtype=np.float64)
        v = np.concatenate([v, pad], axis=-1)
    while v.shape[-1] > 1:
        v = v[..., 0::2] + v[..., 1::2]
    return v[..., 0]


def points(mode: str, K: int, u: float) -> np.ndarray:
    k = np.arange(K, dtype=np.int64)
    if mode == "fp64":
        return (k.astype(np.float64) + np.float64(u)) / np.float64(K)
    if mode == "fp32":
        return ((k.astype(np.float32) + np.float32(u)) / np.float32(K)).astype(np.float64)
    return (k.astype(np.float64) + np.float64(u)) * (1.0 / np.float64(K))


def exp_mode(mode: str, x: np.ndarray) -> np.ndarray:
    if mode == "fp64":
        return rng.exp64_np(x)
    if mode == "fp32":
        return rng.exp32_np(x)
    return exp16_table()[np.asarray(x, dtype=F16).view(np.uint16)]


class FusedTrack:
    """One filter (track) of the fused algorithm."""

    def __init__(self, mode: str, K: int, W: int, H: int, seed: int, start,
                 params: Optional[Params] = None, offsets: Optional[np.ndarray] = None):
        if mode == "fp16-packed":
            mode = "fp16"
        self.mode = mode
        self.d = DT[mode]
        self.K = K
        self.W, self.H = W, H
        self.p = params or Params()
        self.offs = offsets if offsets is not None else disk_offsets(self.p.disk_radius)
        self.r = int(np.max(np.abs(self.offs))) if len(self.offs) else 0
        self.x0 = rng.lcg_seed_state(seed)
        self.n = (K + TILE - 1) // TILE
        self.Q = qbits(self.n)
        d = self.d
        with np.errstate(over="ignore"):
            self.xs = np.full(K, d(start[0]), dtype=d)
            self.ys = np.full(K, d(start[1]), dtype=d)
        self.c = None  # local cdf of previous frame
        self.table = None  # (s, O, invM)
        self.u = None
        self.t = 0
        self.ident = False  # next frame: identity ancestors (injected state)

    def set_state(self, xs: np.ndarray, ys: np.ndarray, t: int) -> None:
        """pf_set_state: post-resample positions entering frame t."""
        with np.errstate(over="ignore"):
            self.xs = np.asarray(xs).astype(self.d)
            self.ys = np.asarray(ys).astype(self.d)
        self.t = int(t)
        self.ident = True

    # -- stages ------------------------------------------------------------
    def ancestors(self) -> np.ndarray:
        K = self.K
        if self.t == 0 or self.ident:
            return np.arange(K, dtype=np.int64)
        s, O, invM = self.table
        k = np.arange(K, dtype=np.int64)
        b = np.searchsorted(s, k, side="right") - 1
        if self.mode == "fp16":
            # f32 tile-local coordinate q = ((k - s_b) + phi_b) * rho_b (table holds phi, rho)
            q = ((k - s[b]).astype(np.float32) + O[b].astype(np.float32)) * invM[b].astype(np.float32)
            q = np.minimum(np.maximum(q, np.float32(0.0)), np.float32(1.0)).astype(np.float64)
        else:
            p = points(self.mode, K, self.u)
            q = (p - O[b]) * invM[b]
            q = np.where(invM[b] == 0.0, 0.0, q)
            q = np.minimum(np.maximum(q, 0.0), 1.0)
        anc = np.empty(K, dtype=np.int64)
        c64 = self.c.astype(np.float64)
        # b is non-decreasing in k: each source tile's outputs are one contiguous run
        tiles = np.unique(b)
        starts = np.searchsorted(b, tiles, side="left")
        ends = np.searchsorted(b, tiles, side="right")
        for tb, k0, k1 in zip(tiles.tolist(), starts.tolist(), ends.tolist()):
            lo = tb * TILE
            hi = min(K, lo + TILE)
            anc[k0:k1] = lo + np.searchsorted(c64[lo:hi], q[k0:k1], side="left")
        return anc

    def propagate(self, anc: np.ndarray, noise: np.ndarray):
        d, p = self.d, self.p
        with np.errstate(over="ignore", invalid="ignore"):
            xa = self.xs[anc]
            ya = self.ys[anc]
            if self.mode == "fp16":
                nx = noise[:, 0].astype(F16)
                ny = noise[:, 1].astype(F16)
                self.xs = ((xa + F16(p.drift_x)).astype(F16) + (F16(p.std_x) * nx).astype(F16)).astype(F16)
                self.ys = ((ya + F16(p.drift_y)).astype(F16) + (F16(p.std_y) * ny).astype(F16)).astype(F16)
            else:
                self.xs = (xa + d(p.drift_x)) + d(p.std_x) * noise[:, 0].astype(d)
                self.ys = (ya + d(p.drift_y)) + d(p.std_y) * noise[:, 1].astype(d)

    def tiles(self, L: np.ndarray):
        """Per-tile max / fixed-point weights / local cdf / moments."""
        K, n, T = self.K, self.n, TILE
        mode, d = self.mode, self.d
        Fb = FBITS[mode]
        pad = n * T - K
        valid = np.concatenate([np.ones(K, bool), np.zeros(pad, bool)]).reshape(n, T)
        Lp = np.concatenate([L.astype(d), np.zeros(pad, dtype=d)]).reshape(n, T)
        with np.errstate(invalid="ignore", over="ignore"):
            neg = d(-np.inf)
            m = np.where(valid, Lp, neg).max(axis=1)
            diff = (Lp - m[:, None]).astype(d)
            w = exp_mode(mode, diff)
            if mode == "fp16":
                wq = np.rint(w.astype(np.float32) * np.float32(2.0**Fb)).astype(np.int64)
            elif mode == "fp32":
                wq = np.rint(w * np.float32(2.0**Fb)).astype(np.int64)
            else:
                wq = np.rint(w * 2.0**Fb).astype(np.int64)
        wq = np.where(valid, wq, 0)
        self.last_wq = wq.reshape(-1)[:K]  # fixed-point tile weights (tests)
        cum = np.cumsum(wq, axis=1)
        S = cum[:, -1]
        if mode == "fp16":
            invf = (np.float32(1.0) / S.astype(np.float32))
            c = (cum.astype(np.float32) * invf[:, None]).astype(F16)
            one = F16(1.0)
        else:
            inv = 1.0 / S.astype(np.float64)
            c = (cum.astype(np.float64) * inv[:, None])
            if mode == "fp32":
                c = c.astype(np.float32)
            one = d(1.0)
        c = np.where(cum == S[:, None], one, c).astype(d)
        xs = np.concatenate([self.xs, np.zeros(pad, dtype=d)]).reshape(n, T)
        ys = np.concatenate([self.ys, np.zeros(pad, dtype=d)]).reshape(n, T)
        if mode == "fp16":
            xq = np.rint(xs.astype(np.float32) * np.float32(2.0**XQ_BITS)).astype(np.int64)
            yq = np.rint(ys.astype(np.float32) * np.float32(2.0**XQ_BITS)).astype(np.int64)
            X = (wq * xq).sum(axis=1)
            Y = (wq * yq).sum(axis=1)
        else:
            wd = wq.astype(np.float64)
            X = pairwise_tree(wd * xs.astype(np.float64), T)
            Y = pairwise_tree(wd * ys.astype(np.float64), T)
        self.c = c.reshape(-1)[:K]
        return m.astype(np.float64), S, X, Y

    def table_step(self, m_b, S, X, Y, u):
        """Tile table (exact prefix) + estimate."""
        n, K = self.n, self.K
        mode = self.mode
        Fb = FBITS[mode]
        m = m_b.max()
        f = rng.exp64_np(m_b - m)
        mass = np.rint((S.astype(np.float64) * f) * 2.0 ** (self.Q - Fb)).astype(np.int64)
        self.last_mass = mass  # exact tile masses (tests)
        Oq = np.concatenate([[0], np.cumsum(mass)[:-1]]).astype(np.int64)
        Sq = int(mass.sum())
        O = Oq.astype(np.float64) / np.float64(Sq)
        with np.errstate(divide="ignore"):
            invM = np.where(mass > 0, np.float64(Sq) / mass.astype(np.float64), 0.0)
        pts = points(mode, K, u)
        s = np.searchsorted(pts, O, side="right").astype(np.int64)
        s[0] = 0
        npad = 1 << int(math.ceil(math.log2(max(1, n))))
        if mode == "fp16":
            nx = pairwise_tree(f * X.astype(np.float64), npad)
            ny = pairwise_tree(f * Y.astype(np.float64), npad)
        else:
            nx = pairwise_tree(f * X, npad)
            ny = pairwise_tree(f * Y, npad)
        den = pairwise_tree(f * S.astype(np.float64), npad)
        ex, ey = float(nx / den), float(ny / den)
        if mode == "fp16":
            ex *= 2.0**-XQ_BITS
            ey *= 2.0**-XQ_BITS
        if mode == "fp16":
            Kd = np.float64(K)
            phi = ((s.astype(np.float64) + np.float64(u)) - Kd * O).astype(np.float32)
            with np.errstate(divide="ignore"):
                rho = np.where(mass > 0, np.float64(Sq) / (Kd * mass.astype(np.float64)), 0.0).astype(np.float32)
            self.table = (s, phi.astype(np.float64), rho.astype(np.float64))
        else:
            self.table = (s, O, invM)
        return ex, ey

    def step(self, Lmap: np.ndarray, noise: Optional[np.ndarray] = None, u: Optional[float] = None
             ) -> Tuple[float, float]:
        """One frame; draws from the LCG stream unless given (noise (K, 2), u),
        e.g. the reference's Generator(Philox(seed)) stream (rng='numpy-philox')."""
        K = self.K
        if noise is None:
            base = self.t * (2 * K + 1)
            words = rng.lcg_words(self.x0, base, 2 * K)
            if self.mode == "fp16":  # precision-matched binary16 draws (rng.normals16_from_lcg_words)
                noise = rng.normals16_from_lcg_words(words).reshape(K, 2)
            else:
                noise = rng.normals_from_lcg_words(words).reshape(K, 2)
            u = (rng.lcg_word(self.x0, base + 2 * K) >> 11) * rng.TWO_M53
        anc = self.ancestors()
        self.last_ancestors = anc
        self.propagate(anc, noise)
        L = lookup(Lmap, self.xs, self.ys, self.W, self.H, self.r)
        self.last_loglik = L
        m_b, S, X, Y = self.tiles(L)
        est = self.table_step(m_b, S, X, Y, u)
        self.u = u
        self.t += 1
        self.ident = False
        return est

    def loglik_map(self, frame: np.ndarray) -> np.ndarray:
        if self.mode == "fp16":
            return loglik_map_half(frame, self.offs, self.p)
        return loglik_map_wide(frame, self.offs, self.p, self.d)


def run(frames: np.ndarray, K: int, mode: str, seed: int, params: Optional[Params] = None,
        offsets: Optional[np.ndarray] = None, start_hint=None, n_frames: Optional[int] = None):
    F, H, W = frames.shape
    if n_frames is not None:
        F = min(F, n_frames)
    if start_hint is None:
        start_hint = (W / 2.0, H / 2.0)
    tr = FusedTrack(mode, K, W, H, seed, start_hint, params, offsets)
    traj = np.empty((F, 2))
    for t in range(F):
        traj[t] = tr.step(tr.loglik_map(frames[t]))
    return traj, tr
