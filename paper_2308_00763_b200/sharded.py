"""Sharded giant filter: one track's particles split by range over shards.

North star (BASELINE.json, config C5): "A single giant filter is sharded by
particle range: an NCCL all-gather of the eight per-shard weight sums and
maxima gives the global normalisation and CDF offsets, and resampled
ancestors that fall outside a shard are fetched peer-to-peer over NVLink."

The reference runs one filter in one process (halfpf.filter.run,
/root/reference/pkg/src/halfpf/filter.py:591-662); its global steps --
max_loglik (:219-220), the weight sum (:228), normalize_and_scan (:233-239),
estimate (:241-246) and resample's CDF search (:248-255) -- are what cross
shards here.  Per frame, on every shard's CUDA stream (include/pf_b200.h):

  pf_shard_fused      resample (peer reads of remote source tiles) ->
                      propagate -> likelihood -> tile weights / local CDF
  all-gather 8 B      shard max keys                  (global max shift)
  pf_shard_tables     exact tile masses, shard total, moment subtree roots
  all-gather 32 B     (mass total, X, Y, D) per shard (offsets, normaliser,
                                                       estimate)
  pf_shard_finish     tile table, source windows written into the owning
                      shards' records (peer stores), estimate
  barrier             windows complete before the next frame reads them

Results are bit-identical to the same filter on one device (Filter / run),
so the shard count never changes a trajectory.

Two exchange back-ends:
  * LocalShards -- S shards as S handles in one process (same or different
    devices), exchanges by device copies + stream events.  This is how the
    sharded path is checked against the single-device filter on one GPU.
  * DistShard   -- one shard per process (torch.distributed, one GPU per rank):
    peer buffers mapped through CUDA IPC, exchanges as all-gathers on the
    library's stream (NCCL); `host_staged=True` stages the tiny payloads
    through host memory instead (gloo), e.g. two processes sharing one GPU.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .filter import DegeneracyError, PrecisionMode, _NATIVE_MODE, _mode, _offsets, _params_struct, _validate_k
from .model import ModelParams, PixelTemplate, disk_template

MAX_SHARDS = 8


def _config(K, mode, width, height, seed, params, template, start_hint, tpb, device):
    mode = _mode(mode)
    _validate_k(K, mode)
    params = params or ModelParams()
    template = template if template is not None else disk_template(params.disk_radius)
    if start_hint is None:
        start_hint = (width / 2.0, height / 2.0)
    seeds = np.asarray([int(seed) & ((1 << 64) - 1)], dtype=np.uint64)
    offs = _offsets(template)
    cfg = N.pf_config()
    cfg.precision = _NATIVE_MODE[mode]
    cfg.K = int(K)
    cfg.width, cfg.height = int(width), int(height)
    cfg.n_tracks, cfg.n_videos = 1, 1
    cfg.seeds = seeds.ctypes.data_as(C.POINTER(C.c_uint64))
    cfg.params = _params_struct(params)
    cfg.offsets_xy = offs.ctypes.data_as(C.POINTER(C.c_int32))
    cfg.n_offsets = template.count
    cfg.tpb = int(tpb or 0)
    cfg.device = int(device)
    cfg.start_x, cfg.start_y = float(start_hint[0]), float(start_hint[1])
    return cfg, (seeds, offs)  # keep the arrays alive while the config is used


def shard_layout(K: int, n_shards: int, tile: int = 1024) -> Tuple[int, List[Tuple[int, int]]]:
    """(tiles per shard, [(first particle, count)] per shard) -- mirrors pf_shard_create."""
    n_tiles = -(-K // tile)
    per = -(-n_tiles // n_shards)
    st = 1
    while st < per:
        st <<= 1
    if (n_shards - 1) * st >= n_tiles:
        raise ValueError("too few tiles for this many shards (every shard must hold particles)")
    out = []
    for r in range(n_shards):
        first = r * st * tile
        out.append((first, min(K, first + st * tile) - first))
    return st, out


class _Shard:
    """One shard handle (one GPU's particle range)."""

    def __init__(self, K, mode, width, height, seed, n_shards, shard, params=None, template=None,
                 start_hint=None, tpb=None, device=0):
        if not 2 <= n_shards <= MAX_SHARDS:
            raise ValueError(f"n_shards must be in [2, {MAX_SHARDS}]")
        self.mode = _mode(mode)
        self.K, self.n_shards, self.shard = int(K), int(n_shards), int(shard)
        self.width, self.height = int(width), int(height)
        cfg, keep = _config(K, mode, width, height, seed, params, template, start_hint, tpb, device)
        L = N.lib()
        h = C.c_void_p()
        rc = L.pf_shard_create(C.byref(h), C.byref(cfg), self.n_shards, self.shard)
        if rc == N.PF_EINVAL:
            raise ValueError(L.pf_global_error().decode())
        N.check(rc, L.pf_global_error)
        del keep
        self._h = h
        self.device = device
        info = np.zeros(4, dtype=np.int64)
        N.check(L.pf_shard_info(h, N.ptr(info)), self._err)
        self.shard_tiles, self.tile0, self.n_local, self.K_local = (int(v) for v in info)

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

    def buffers(self) -> List[int]:
        out = (C.c_void_p * 8)()
        N.check(N.lib().pf_shard_buffers(self._h, out), self._err)
        return [int(v or 0) for v in out]

    def ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(8 * 64)
        N.check(N.lib().pf_shard_ipc_export(self._h, buf), self._err)
        return buf.raw

    def set_peer(self, peer: int, ptrs: Sequence[int]):
        arr = (C.c_void_p * 8)(*[C.c_void_p(p) for p in ptrs])
        N.check(N.lib().pf_shard_set_peer(self._h, int(peer), arr), self._err)

    def open_peer(self, peer: int, handles: bytes):
        buf = C.create_string_buffer(handles, len(handles))
        N.check(N.lib().pf_shard_open_peer(self._h, int(peer), buf), self._err)

    def exchange(self) -> List[int]:
        out = (C.c_void_p * 4)()
        N.check(N.lib().pf_shard_exchange(self._h, out), self._err)
        return [int(v) for v in out]

    def stream(self) -> int:
        return int(N.lib().pf_shard_stream(self._h) or 0)

    def reset(self, start_hint):
        N.check(N.lib().pf_reset(self._h, float(start_hint[0]), float(start_hint[1])), self._err)

    def begin(self, frames):
        if hasattr(frames, "data_ptr") and getattr(frames, "is_cuda", False):
            self._keep = frames
            N.check(N.lib().pf_shard_begin(self._h, C.c_void_p(frames.data_ptr()), int(frames.shape[0]), 1),
                    self._err)
        else:
            arr = np.ascontiguousarray(np.asarray(frames, dtype=np.uint8))
            self._keep = arr
            N.check(N.lib().pf_shard_begin(self._h, N.ptr(arr), int(arr.shape[0]), 0), self._err)

    def fused(self, f: int):
        N.check(N.lib().pf_shard_fused(self._h, int(f)), self._err)

    def tables(self):
        N.check(N.lib().pf_shard_tables(self._h), self._err)

    def finish(self, f: int):
        N.check(N.lib().pf_shard_finish(self._h, int(f)), self._err)

    def end(self, F: int) -> np.ndarray:
        traj = np.empty((F, 2), dtype=np.float64)
        rc = N.lib().pf_shard_end(self._h, int(F), N.ptr(traj))
        if rc == N.PF_EDEGENERATE:
            raise DegeneracyError(self._err().decode(), N.lib().pf_degenerate_frame(self._h))
        N.check(rc, self._err)
        self._keep = None
        return traj

    def timings(self):
        t = (C.c_float * 6)()
        N.check(N.lib().pf_last_timings(self._h, t), self._err)
        return float(t[0])


class LocalShards:
    """S shards of one filter held by one process (devices may repeat).

    `run(frames)` returns the (F, 2) trajectory, bit-identical to
    `Filter(K, ...).run(frames)`.
    """

    def __init__(self, K: int, mode="fp16", width: int = 128, height: int = 128, seed: int = 42,
                 n_shards: int = 2, params: Optional[ModelParams] = None,
                 template: Optional[PixelTemplate] = None, start_hint=None, tpb=None,
                 devices: Optional[Sequence[int]] = None):
        devices = list(devices) if devices is not None else [0] * n_shards
        if len(devices) != n_shards:
            raise ValueError("one device per shard")
        self.start_hint = start_hint if start_hint is not None else (width / 2.0, height / 2.0)
        self.shards = [_Shard(K, mode, width, height, seed, n_shards, r, params, template, self.start_hint, tpb,
                              devices[r]) for r in range(n_shards)]
        bufs = [s.buffers() for s in self.shards]
        for s in self.shards:
            for q, b in enumerate(bufs):
                if q != s.shard:
                    s.set_peer(q, b)
        self._arr = (C.c_void_p * n_shards)(*[s._h for s in self.shards])

    def _gather(self, which: int):
        N.check(N.lib().pf_shard_local_allgather(self._arr, len(self.shards), which), self.shards[0]._err)

    def reset(self, start_hint=None):
        if start_hint is not None:
            self.start_hint = start_hint
        for s in self.shards:
            s.reset(self.start_hint)

    def run(self, frames) -> np.ndarray:
        F = int(frames.shape[0])
        for s in self.shards:
            s.begin(frames)
        for f in range(F):
            for s in self.shards:
                s.fused(f)
            self._gather(0)
            for s in self.shards:
                s.tables()
            self._gather(1)
            for s in self.shards:
                s.finish(f)
            self._gather(2)
        trajs = [s.end(F) for s in self.shards]
        for t in trajs[1:]:  # every shard computes the same estimate
            if not np.array_equal(t, trajs[0]):
                raise RuntimeError("shards disagree on the estimate")
        return trajs[0]

    def close(self):
        for s in self.shards:
            s.close()


class _DevArray:
    """Zero-copy view of a library device buffer for torch (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class DistShard:
    """This process's shard of one filter (torch.distributed, one rank per shard).

    Peer buffers are mapped through CUDA IPC (handles exchanged with
    all_gather_object).  The per-frame exchanges are all-gathers issued on the
    library's stream (NCCL over NVLink); with `host_staged=True` the 8 / 32 B
    payloads go through host memory (gloo), which also works for ranks that
    share a GPU.
    """

    def __init__(self, K: int, mode="fp16", width: int = 128, height: int = 128, seed: int = 42,
                 params=None, template=None, start_hint=None, tpb=None, device: int = 0,
                 host_staged: bool = False, dist=None):
        import torch
        import torch.distributed as tdist

        self.dist = dist or tdist
        self.torch = torch
        self.world = self.dist.get_world_size()
        self.rank = self.dist.get_rank()
        self.host_staged = host_staged
        self.start_hint = start_hint if start_hint is not None else (width / 2.0, height / 2.0)
        self.s = _Shard(K, mode, width, height, seed, self.world, self.rank, params, template, self.start_hint,
                        tpb, device)
        handles = [None] * self.world
        self.dist.all_gather_object(handles, self.s.ipc_handles())
        for q, hb in enumerate(handles):
            if q != self.rank:
                self.s.open_peer(q, hb)
        ex = self.s.exchange()
        dev = torch.device("cuda", device)
        self.max_send = torch.as_tensor(_DevArray(ex[0], 1, "<i8"), device=dev)
        self.max_recv = torch.as_tensor(_DevArray(ex[1], self.world, "<i8"), device=dev)
        self.sum_send = torch.as_tensor(_DevArray(ex[2], 4, "<i8"), device=dev)
        self.sum_recv = torch.as_tensor(_DevArray(ex[3], 4 * self.world, "<i8"), device=dev)
        self.token = torch.zeros(1, dtype=torch.int32, device=dev)
        self.token_recv = torch.zeros(self.world, dtype=torch.int32, device=dev)
        self.stream = torch.cuda.ExternalStream(self.s.stream(), device=dev)

    def _allgather(self, recv, send):
        if self.host_staged:
            self.stream.synchronize()
            parts = [self.torch.empty_like(send, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, send.cpu())
            recv.copy_(self.torch.cat(parts).to(recv.device))
            self.torch.cuda.current_stream(recv.device).synchronize()
        else:
            with self.torch.cuda.stream(self.stream):
                self.dist.all_gather_into_tensor(recv, send)

    def reset(self, start_hint=None):
        if start_hint is not None:
            self.start_hint = start_hint
        self.s.reset(self.start_hint)

    def run(self, frames) -> np.ndarray:
        F = int(frames.shape[0])
        self.s.begin(frames)
        for f in range(F):
            self.s.fused(f)
            self._allgather(self.max_recv, self.max_send)
            self.s.tables()
            self._allgather(self.sum_recv, self.sum_send)
            self.s.finish(f)
            self._allgather(self.token_recv, self.token)  # barrier: windows written everywhere
        return self.s.end(F)

    def close(self):
        self.s.close()
