"""ORACLE (test infrastructure only) -- host restatement of the draw streams.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.  Nothing here is on the product path.

Two streams are restated:

1. The reference stream, `RngStream` (/root/reference/pkg/src/halfpf/filter.py:71-82):
   `Generator(Philox(seed))`; `normals(K)` = `standard_normal((K, 2))`
   (C order: particle k takes one normal for x then one for y), `uniform()` =
   `random()` = `(word >> 11) * 2**-53`.  `standard_normal` is NumPy's
   256-layer ziggurat (numpy/random/src/distributions/distributions.c,
   `random_standard_normal`; tables from oracle/ziggurat_tables.npz).  The
   word source is NumPy's own `Philox.random_raw`, so this restatement pins
   the ziggurat tables and the normal transform bit-exactly
   (tests/test_oracle_rng.py).

2. The product stream ("lcg", the north star's counter-based LCG): one
   64-bit MMIX LCG sequence per seed, x_{n+1} = A*x_n + C (mod 2^64),
   x_0 = splitmix64(seed).  Word n is x_n.  Frame t of a K-particle filter
   consumes positions t*(2K+1) + 2k + c for the normals (particle k,
   component c) and t*(2K+1) + 2K for the resampling uniform -- exactly the
   order in which `run()` calls `normals(K)` then `uniform()`, so an
   `LcgStream` injected in place of `RngStream` feeds the reference the same
   draws the device generates.  The normal transform is the same ziggurat
   with the layer index, sign and 52-bit magnitude taken from the HIGH bits
   (idx = r>>56, sign = bit 55, rabs = bits 3..54) because the low bits of a
   power-of-two LCG are weak; the rare slow path (about 1.2% of normals)
   draws its extra words from a splitmix64 sequence seeded with the primary
   word, so every normal is a pure function of its stream position.  exp and
   log1p in the slow path are the portable IEEE-only restatements below, so
   the device reproduces every draw bit-exactly.
"""

from __future__ import annotations

import os

import numpy as np

M64 = (1 << 64) - 1
LCG_A = 6364136223846793005
LCG_C = 1442695040888963407
GOLDEN = 0x9E3779B97F4A7C15
ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828
TWO_M53 = 1.0 / 9007199254740992.0
MASK52 = (1 << 52) - 1

_T = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ziggurat_tables.npz"))
KI = [int(v) for v in _T["ki"]]
WI = [float(v) for v in _T["wi"]]
FI = [float(v) for v in _T["fi"]]
KI_NP = _T["ki"].astype(np.uint64)
WI_NP = _T["wi"].astype(np.float64)


# --------------------------------------------------------------------------
# portable IEEE-only exp / log1p (the device compiles the same op sequence
# with __dadd_rn/__dmul_rn, so results are bit-identical by construction)
# --------------------------------------------------------------------------

LOG2E = 1.4426950408889634
LN2_HI = 6.93147180369123816490e-01
LN2_LO = 1.90821492927058770002e-10
_EXP_C = [1.0]
for _i in range(1, 14):
    _EXP_C.append(_EXP_C[-1] / _i)  # 1/i!, each rounded once more -- fixed constants
EXP_COEF = [float(c) for c in _EXP_C]  # c0..c13
SQRT2 = 1.4142135623730951
LOG_COEF = [1.0 / (2 * i + 1) for i in range(12)]  # 1, 1/3, ..., 1/23


def _pow2(k: int) -> float:
    return float(np.uint64((k + 1023) << 52).view(np.float64))


def exp64(x: float) -> float:
    """Portable exp: Cody-Waite reduction + degree-13 Taylor (Horner)."""
    x = float(x)
    if x != x:
        return x
    if x < -708.0:
        return 0.0
    if x > 709.0:
        return float("inf")
    k = float(np.rint(x * LOG2E))
    r = (x - k * LN2_HI) - k * LN2_LO
    p = EXP_COEF[13]
    for i in range(12, -1, -1):
        p = p * r + EXP_COEF[i]
    return p * _pow2(int(k))


def exp64_np(x: np.ndarray) -> np.ndarray:
    """Vectorised exp64 (identical op sequence)."""
    x = np.asarray(x, dtype=np.float64)
    xc = np.clip(x, -708.0, 709.0)
    k = np.rint(xc * LOG2E)
    r = (xc - k * LN2_HI) - k * LN2_LO
    p = np.full_like(r, EXP_COEF[13])
    for i in range(12, -1, -1):
        p = p * r + EXP_COEF[i]
    scale = ((k.astype(np.int64) + 1023) << 52).astype(np.uint64).view(np.float64)
    out = p * scale
    out = np.where(x < -708.0, 0.0, out)
    out = np.where(x > 709.0, np.inf, out)
    return np.where(np.isnan(x), x, out)


def log64(u: float) -> float:
    """Portable log for finite u > 0 (normal range)."""
    bits = int(np.float64(u).view(np.uint64))
    e = ((bits >> 52) & 0x7FF) - 1023
    m = float(np.uint64((bits & MASK52) | (1023 << 52)).view(np.float64))
    if m > SQRT2:
        m = m * 0.5
        e += 1
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    p = LOG_COEF[11]
    for i in range(10, -1, -1):
        p = p * z + LOG_COEF[i]
    logm = (s + s) * p
    ef = float(e)
    return ef * LN2_HI + (ef * LN2_LO + logm)


def log1p64(x: float) -> float:
    """Portable log1p for x > -1 (Goldberg's u = 1 + x correction)."""
    u = 1.0 + x
    if u == 1.0:
        return x
    return log64(u) * (x / (u - 1.0))


# f32 portable exp (fused FP32 weights)
LN2_HI_F = np.float32(0.693145751953125)
LN2_LO_F = np.float32(1.428606765330187045e-06)
LOG2E_F = np.float32(1.4426950408889634)
EXPF_COEF = [np.float32(c) for c in EXP_COEF[:9]]  # c0..c8


def exp32_np(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    xc = np.clip(x, np.float32(-87.0), np.float32(88.0))
    k = np.rint(xc * LOG2E_F)
    r = (xc - k * LN2_HI_F) - k * LN2_LO_F
    p = np.full_like(r, EXPF_COEF[8])
    for i in range(7, -1, -1):
        p = p * r + EXPF_COEF[i]
    scale = ((k.astype(np.int32) + 127) << 23).astype(np.uint32).view(np.float32)
    out = p * scale
    out = np.where(x < np.float32(-87.0), np.float32(0.0), out)
    out = np.where(x > np.float32(88.0), np.float32(np.inf), out)
    return np.where(np.isnan(x), x, out).astype(np.float32)


# --------------------------------------------------------------------------
# integer helpers
# --------------------------------------------------------------------------


def splitmix64_mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def lcg_seed_state(seed: int) -> int:
    """x_0 = splitmix64(seed) (one splitmix step from state `seed`)."""
    return splitmix64_mix((int(seed) + GOLDEN) & M64)


def affine_pow(n: int, a: int = LCG_A, c: int = LCG_C):
    """(A_n, C_n) with x_{m+n} = A_n * x_m + C_n (mod 2^64)."""
    ra, rc = 1, 0
    ba, bc = a, c
    while n:
        if n & 1:
            # apply base after current: x -> ba*(ra*x+rc)+bc
            ra, rc = (ba * ra) & M64, (ba * rc + bc) & M64
        ba, bc = (ba * ba) & M64, (ba * bc + bc) & M64
        n >>= 1
    return ra, rc


def lcg_word(x0: int, n: int) -> int:
    a, c = affine_pow(n)
    return (a * x0 + c) & M64


def lcg_words(x0: int, start: int, count: int) -> np.ndarray:
    """Words [start, start+count) of the stream, vectorised."""
    a0, c0 = affine_pow(start)
    xs = (a0 * x0 + c0) & M64
    out = np.empty(count, dtype=np.uint64)
    if count == 0:
        return out
    # doubling: a[i], c[i] for f^i
    a = np.ones(1, dtype=np.uint64)
    c = np.zeros(1, dtype=np.uint64)
    m = 1
    am, cm = LCG_A, LCG_C
    while m < count:
        am_u, cm_u = np.uint64(am), np.uint64(cm)
        a2 = a * am_u
        c2 = a * cm_u + c
        a = np.concatenate([a, a2])
        c = np.concatenate([c, c2])
        am, cm = (am * am) & M64, (am * cm + cm) & M64
        m *= 2
    a = a[:count]
    c = c[:count]
    with np.errstate(over="ignore"):
        out[:] = a * np.uint64(xs) + c
    return out


class _Retry:
    """splitmix64 sequence seeded with the primary word (slow-path draws)."""

    def __init__(self, w: int):
        self.s = w

    def next64(self) -> int:
        self.s = (self.s + GOLDEN) & M64
        return splitmix64_mix(self.s)

    def next_double(self) -> float:
        return (self.next64() >> 11) * TWO_M53


def _zig_slow_lcg(r: int) -> float:
    """Full ziggurat for primary word r (LCG high-bit layout); slow path."""
    retry = _Retry(r)
    while True:
        idx = r >> 56
        sign = (r >> 55) & 1
        rabs = (r >> 3) & MASK52
        x = float(rabs) * WI[idx]
        if sign:
            x = -x
        if rabs < KI[idx]:
            return x
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * log1p64(-retry.next_double())
                yy = -log1p64(-retry.next_double())
                if yy + yy > xx * xx:
                    return -(ZIG_R + xx) if sign else ZIG_R + xx
        else:
            if (FI[idx - 1] - FI[idx]) * retry.next_double() + FI[idx] < exp64(-0.5 * x * x):
                return x
        r = retry.next64()


def normals_from_lcg_words(words: np.ndarray) -> np.ndarray:
    """One normal per primary word (fast path vectorised)."""
    w = words.astype(np.uint64)
    idx = (w >> np.uint64(56)).astype(np.int64)
    sign = ((w >> np.uint64(55)) & np.uint64(1)).astype(bool)
    rabs = (w >> np.uint64(3)) & np.uint64(MASK52)
    x = rabs.astype(np.float64) * WI_NP[idx]
    x = np.where(sign, -x, x)
    slow = ~(rabs < KI_NP[idx])
    for i in np.nonzero(slow)[0]:
        x[i] = _zig_slow_lcg(int(w[i]))
    return x


# binary16 modes of the fused kernels ("precision-matched" draws): the same
# word stream, the ziggurat fast path evaluated in binary32 on the word's high
# 32 bits -- idx = bits 56..63, sign = bit 55, rabs = bits 32..54 (23 bits) --
# with tables ki32 = ki >> 29 and wi32 = RN32(wi * 2^29); x = RN32(rabs * wi32),
# then RN16.  A word failing the binary32 fast test takes the full f64 slow
# path of the same word (_zig_slow_lcg), rounded once to binary16.
KI32_NP = (KI_NP >> np.uint64(29)).astype(np.uint32)
WI32_NP = (WI_NP * 2.0**29).astype(np.float32)


def normals16_from_lcg_words(words: np.ndarray) -> np.ndarray:
    """One binary16 normal per primary word (fused FP16 / FP16-packed draws)."""
    w = words.astype(np.uint64)
    hi = (w >> np.uint64(32)).astype(np.uint32)
    idx = (hi >> np.uint32(24)).astype(np.int64)
    sign = ((hi >> np.uint32(23)) & np.uint32(1)).astype(bool)
    rabs = hi & np.uint32(0x7FFFFF)
    x = rabs.astype(np.float32) * WI32_NP[idx]  # one binary32 RN multiply
    x = np.where(sign, -x, x)
    out = x.astype(np.float16)
    for i in np.nonzero(~(rabs < KI32_NP[idx]))[0]:
        out[i] = np.float16(_zig_slow_lcg(int(w[i])))
    return out


class LcgStream:
    """Drop-in `RngStream` replacement (same methods) emitting the LCG stream."""

    def __init__(self, seed: int):
        self.seed = seed
        self.x0 = lcg_seed_state(seed)
        self.pos = 0

    def normals(self, n: int) -> np.ndarray:
        w = lcg_words(self.x0, self.pos, 2 * n)
        self.pos += 2 * n
        return normals_from_lcg_words(w).reshape(n, 2)

    def uniform(self) -> float:
        w = lcg_word(self.x0, self.pos)
        self.pos += 1
        return (w >> 11) * TWO_M53


def frame_draws(seed: int, K: int, t: int):
    """(normals (K,2), u) of frame t, by stream position (no state)."""
    x0 = lcg_seed_state(seed)
    base = t * (2 * K + 1)
    w = lcg_words(x0, base, 2 * K)
    u = (lcg_word(x0, base + 2 * K) >> 11) * TWO_M53
    return normals_from_lcg_words(w).reshape(K, 2), u


# --------------------------------------------------------------------------
# NumPy layout (reference stream) -- used to pin the tables
# --------------------------------------------------------------------------


class _WordSource:
    def __init__(self, words):
        self.w = [int(v) for v in words]
        self.i = 0

    def next64(self) -> int:
        v = self.w[self.i]
        self.i += 1
        return v

    def next_double(self) -> float:
        return (self.next64() >> 11) * TWO_M53


# --------------------------------------------------------------------------
# glibc 2.39 x86-64 log1p (FMA ifunc variant), restated from its disassembly:
# NumPy's ziggurat tail calls npy_log1p == glibc log1p, so the reference
# stream's rare tail normals depend on it bit-for-bit.  fma() is exact
# (Fraction) here and __fma_rn on the device.
# --------------------------------------------------------------------------

def _fma(a: float, b: float, c: float) -> float:
    from fractions import Fraction

    return float(Fraction(a) * Fraction(b) + Fraction(c))


_G_L1, _G_L2, _G_L3 = float.fromhex("0x1.5555555555593p-1"), float.fromhex("0x1.999999997fa04p-2"), \
    float.fromhex("0x1.2492494229359p-2")
_G_L4, _G_L5 = float.fromhex("0x1.c71c51d8e78afp-3"), float.fromhex("0x1.7466496cb03dep-3")
_G_L6, _G_L7 = float.fromhex("0x1.39a09d078c69fp-3"), float.fromhex("0x1.2f112df3e5244p-3")
_G_LN2_LO, _G_LN2_HI = float.fromhex("0x1.a39ef35793c76p-33"), float.fromhex("0x1.62e42fee00000p-1")
_G_C23 = float.fromhex("0x1.5555555555555p-1")


def _bits(x: float) -> int:
    return int(np.float64(x).view(np.uint64))


def _frombits(b: int) -> float:
    return float(np.uint64(b).view(np.float64))


def log1p_glibc(x: float) -> float:
    """glibc log1p for -1 < x <= 0.41422 (the ziggurat tail domain)."""
    hx = _bits(x) >> 32
    hx = hx - (1 << 32) if hx & 0x80000000 else hx
    ax = hx & 0x7FFFFFFF
    if ax <= 0x3E1FFFFF:
        if ax <= 0x3C8FFFFF:
            return x
        return _fma(-(x * x), 0.5, x)
    c = 0.0
    if ((hx + 0x402D413C) & 0xFFFFFFFF) > 0x402D413C:
        k, f, hu = 0, x, 1
    else:
        u = 1.0 + x
        hu = _bits(u) >> 32
        k = (hu >> 20) - 1023
        c = (1.0 - (u - x)) if k > 0 else (x - (u - 1.0))
        c = c / u
        hu &= 0xFFFFF
        lo = _bits(u) & 0xFFFFFFFF
        if hu > 0x6A09D:
            k += 1
            u = _frombits(((hu | 0x3FE00000) << 32) | lo)
            hu = (0x100000 - hu) >> 2
        else:
            u = _frombits(((hu | 0x3FF00000) << 32) | lo)
        f = u - 1.0
    hfsq = (f * 0.5) * f
    kf = float(k)
    if hu == 0:
        if f == 0.0:
            return 0.0 if k == 0 else _fma(kf, _G_LN2_HI, _fma(kf, _G_LN2_LO, c))
        R = _fma(-f, _G_C23, 1.0) * hfsq
        if k == 0:
            return f - R
        return _fma(kf, _G_LN2_HI, -((R - _fma(kf, _G_LN2_LO, c)) - f))
    s = f / (f + 2.0)
    z = s * s
    t11 = _fma(z, _G_L3, _G_L2)
    t10 = _fma(z, _G_L5, _G_L4)
    t9 = _fma(z, _G_L7, _G_L6)
    z2 = z * z
    z4 = z2 * z2
    z6 = z2 * z4
    R = _fma(z6, t9, _fma(z4, t10, _fma(z, _G_L1, z2 * t11)))
    t = (R + hfsq) * s
    if k == 0:
        return f - (hfsq - t)
    klo = _fma(kf, _G_LN2_LO, c)
    return _fma(kf, _G_LN2_HI, -((hfsq - (klo + t)) - f))


def numpy_standard_normal(src: _WordSource, libm_exp=None, libm_log1p=None) -> float:
    """random_standard_normal (distributions.c) over a raw word source.

    The slow path uses libm exp/log1p (math.exp / math.log1p = glibc, the
    same libm NumPy links)."""
    import math

    ex = libm_exp or math.exp
    l1p = libm_log1p or log1p_glibc
    while True:
        r = src.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & MASK52
        x = float(rabs) * WI[idx]
        if sign & 1:
            x = -x
        if rabs < KI[idx]:
            return x
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * l1p(-src.next_double())
                yy = -l1p(-src.next_double())
                if yy + yy > xx * xx:
                    return -(ZIG_R + xx) if ((rabs >> 8) & 1) else ZIG_R + xx
        else:
            if (FI[idx - 1] - FI[idx]) * src.next_double() + FI[idx] < ex(-0.5 * x * x):
                return x
