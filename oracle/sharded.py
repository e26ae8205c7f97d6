"""ORACLE (test infrastructure only) -- the sharded giant filter's exchange
protocol restated on the CPU (paper_2308_00763_b200/sharded.py, the
pf_shard_* kernels in csrc/pf_kernels.cuh).

Each shard holds a particle range of one filter (oracle/fused.py's tile
algorithm); per frame it exchanges, through `comm.allgather(obj)`:
  1. its max tile log-likelihood                    (8 B per shard on the GPU)
  2. its exact int64 mass total and the canonical pairwise subtree roots of
     its tiles' estimate moments                    (32 B per shard)
  3. (peer reads on the GPU) its table entries, local CDF and positions, for
     the shards whose outputs resample from it -- gathered wholesale here.
The composition equals oracle.fused.run on the whole filter bit-for-bit
(tiles per shard are a power of two, so each shard's subtree root is a node of
the global tree); tests/test_multiproc.py checks that with gloo.
"""

from __future__ import annotations

import math

import numpy as np

from . import rng
from .fused import DT, FBITS, TILE, XQ_BITS, FusedTrack, pairwise_tree, points, qbits


def shard_tiles(K: int, n_shards: int) -> int:
    n = -(-K // TILE)
    st = 1 << max(0, math.ceil(math.log2(-(-n // n_shards))))
    if (n_shards - 1) * st >= n:
        raise ValueError("too few tiles for this many shards")
    return st


class ShardTrack:
    def __init__(self, mode, K, W, H, seed, start, shard, n_shards, comm, params=None, offsets=None):
        self.full = FusedTrack(mode, K, W, H, seed, start, params, offsets)  # global constants, map builder
        self.mode, self.K = self.full.mode, K
        self.shard, self.S, self.comm = shard, n_shards, comm
        self.st = shard_tiles(K, n_shards)
        self.n = self.full.n
        self.t0 = shard * self.st
        self.nl = min(self.n - self.t0, self.st)
        self.k0 = self.t0 * TILE
        self.Kl = min(K, self.k0 + self.nl * TILE) - self.k0
        d = self.full.d
        with np.errstate(over="ignore"):
            self.xs = np.full(self.Kl, d(start[0]), dtype=d)
            self.ys = np.full(self.Kl, d(start[1]), dtype=d)
        self.glob = None  # gathered previous-frame (s, O, invM, c, xs, ys)
        self.u = None
        self.t = 0

    def _ancestors(self):
        if self.t == 0:
            return np.arange(self.k0, self.k0 + self.Kl, dtype=np.int64)
        s, O, invM, c, _, _ = self.glob
        k = np.arange(self.k0, self.k0 + self.Kl, dtype=np.int64)
        b = np.searchsorted(s, k, side="right") - 1
        if self.mode == "fp16":
            q = ((k - s[b]).astype(np.float32) + O[b].astype(np.float32)) * invM[b].astype(np.float32)
            q = np.minimum(np.maximum(q, np.float32(0.0)), np.float32(1.0)).astype(np.float64)
        else:
            p = points(self.mode, self.K, self.u)[k]
            q = np.where(invM[b] == 0.0, 0.0, (p - O[b]) * invM[b])
            q = np.minimum(np.maximum(q, 0.0), 1.0)
        anc = np.empty(self.Kl, dtype=np.int64)
        c64 = c.astype(np.float64)
        for tb in np.unique(b):
            sel = b == tb
            lo, hi = tb * TILE, min(self.K, tb * TILE + TILE)
            anc[sel] = lo + np.searchsorted(c64[lo:hi], q[sel], side="left")
        return anc

    def step(self, Lmap):
        full, K, mode = self.full, self.K, self.mode
        base = self.t * (2 * K + 1)
        words = rng.lcg_words(full.x0, base + 2 * self.k0, 2 * self.Kl)
        noise = rng.normals_from_lcg_words(words).reshape(self.Kl, 2)
        u = (rng.lcg_word(full.x0, base + 2 * K) >> 11) * rng.TWO_M53
        anc = self._ancestors()
        if self.t > 0:  # peer reads of the ancestors' positions
            _, _, _, _, gx, gy = self.glob
            full.xs, full.ys = gx, gy
        else:
            full.xs, full.ys = self.xs, self.ys
            anc = anc - self.k0
        full.propagate(anc, noise)
        self.xs, self.ys = full.xs, full.ys
        from .reference_port import lookup

        L = lookup(Lmap, self.xs, self.ys, full.W, full.H, full.r)
        # local tiles (FusedTrack.tiles on this shard's range)
        full_K, full_n = full.K, full.n
        full.K, full.n = self.Kl, self.nl
        m_b, S, X, Y = full.tiles(L)
        c_local = full.c
        full.K, full.n = full_K, full_n
        # exchange 1: max
        m = max(self.comm.allgather(float(m_b.max())))
        Fb = FBITS[mode]
        f = rng.exp64_np(m_b - m)
        mass = np.rint((S.astype(np.float64) * f) * 2.0 ** (qbits(self.n) - Fb)).astype(np.int64)
        Xd = X.astype(np.float64) if mode == "fp16" else X
        Yd = Y.astype(np.float64) if mode == "fp16" else Y
        roots = (pairwise_tree(f * Xd, self.st), pairwise_tree(f * Yd, self.st),
                 pairwise_tree(f * S.astype(np.float64), self.st))
        # exchange 2: (mass total, subtree roots)
        got = self.comm.allgather((int(mass.sum()), [float(v) for v in roots]))
        offset = sum(g[0] for g in got[: self.shard])
        Sq = sum(g[0] for g in got)
        w = 1 << max(0, math.ceil(math.log2(self.S)))
        tree = [pairwise_tree(np.array([g[1][i] for g in got]), w) for i in range(3)]
        ex, ey = float(tree[0] / tree[2]), float(tree[1] / tree[2])
        if mode == "fp16":
            ex *= 2.0**-XQ_BITS
            ey *= 2.0**-XQ_BITS
        Oq = offset + np.concatenate([[0], np.cumsum(mass)[:-1]]).astype(np.int64)
        O = Oq.astype(np.float64) / np.float64(Sq)
        with np.errstate(divide="ignore"):
            invM = np.where(mass > 0, np.float64(Sq) / mass.astype(np.float64), 0.0)
        pts = points(mode, K, u)
        s = np.searchsorted(pts, O, side="right").astype(np.int64)
        if self.shard == 0:
            s[0] = 0
        if mode == "fp16":
            Kd = np.float64(K)
            phi = ((s.astype(np.float64) + np.float64(u)) - Kd * O).astype(np.float32).astype(np.float64)
            with np.errstate(divide="ignore"):
                rho = np.where(mass > 0, np.float64(Sq) / (Kd * mass.astype(np.float64)), 0.0)
            O, invM = phi, rho.astype(np.float32).astype(np.float64)
        # exchange 3 (peer reads on the GPU): table entries, local CDFs, positions
        parts = self.comm.allgather((s, O, invM, c_local, self.xs, self.ys))
        self.glob = tuple(np.concatenate([p[i] for p in parts]) for i in range(6))
        self.u = u
        self.t += 1
        return ex, ey


def run_shard(frames, K, mode, seed, shard, n_shards, comm, start_hint=None):
    F, H, W = frames.shape
    if start_hint is None:
        start_hint = (W / 2.0, H / 2.0)
    tr = ShardTrack(mode, K, W, H, seed, start_hint, shard, n_shards, comm)
    traj = np.empty((F, 2))
    for t in range(F):
        traj[t] = tr.step(tr.full.loglik_map(frames[t]))
    return traj
