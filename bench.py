#!/usr/bin/env python
"""bench.py -- particle-updates/s of the fused per-frame tracking step on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

A "step" is one full tracking run over the config's synthetic video (every
frame: resample -> propagate -> likelihood -> weights -> exact scan / local
CDF -> estimate, plus the per-frame likelihood maps), i.e. K*F particle-
updates per track.  Default config C2 (BASELINE.json configs[1]): 128x128,
100 frames, 1M particles, stabilised FP16 (FP32 / FP64 measured alongside).
With N GPUs (torchrun) every rank runs its own independent track(s) -- the
batched-track sharding of the north star, no collective on the data path
(weak scaling).  Timing: device CUDA events recorded by the library on its
own stream, L2 flushed (512 MiB write) before every timed step, max over
ranks.  `e2e` re-times the same steps through the host-buffer C-ABI call
(frames H2D + trajectory D2H inside the region, wall clock).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-updates/sec (N×frames/s) fp16/fp32/fp64 at 1–8 B200; tracking RMSE"
UNIT = "particle-updates/s"
SIZES = {"fp64": 8, "fp32": 4, "fp16": 2, "fp16-packed": 2}
DTYPE_TAG = {"fp64": "f64", "fp32": "f32", "fp16": "f16", "fp16-packed": "f16"}

CONFIGS = {
    "c1": dict(W=128, H=128, F=10, K=10_000, precision="fp64", tracks=1, videos=1,
               desc="C1: 128x128 video, 10 frames, 10,000 particles, FP64"),
    "c2": dict(W=128, H=128, F=100, K=1_000_000, precision="fp16-packed", tracks=1, videos=1,
               desc="C2: 128x128 video, 100 frames, 1M particles, stabilised FP16 in half2 lanes "
                    "(scalar-lane FP16, FP32, FP64 alongside)"),
    "c3": dict(W=1024, H=1024, F=100, K=1 << 24, precision="fp16-packed", tracks=1, videos=1,
               desc="C3: 1024x1024 video, 100 frames, 16M particles, FP16 half2"),
    "c4": dict(W=128, H=128, F=100, K=65536, precision="fp16-packed", tracks=8192, videos=8,
               desc="C4: 8192 independent 128x128 tracks x 64K particles, FP16 (tracks split over GPUs)"),
    "c5": dict(W=1024, H=1024, F=10, K=1 << 30, precision="fp16-packed", tracks=1, videos=1, sharded=True,
               desc="C5: one 2^30-particle FP16 filter, 1024x1024 video, 10 frames, particle range sharded "
                    "over the GPUs (NCCL all-gathers of shard max / sums, peer reads of remote ancestors)"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 10 ms) during the timed region."""

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self._stop = threading.Event()
        self.thread = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            self.mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            self.thread = None
            return

        def loop():
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
            while not self._stop.is_set():
                try:
                    clk = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((clk, [n for n, b in bits.items() if r & b]))
                except Exception:
                    pass
                time.sleep(0.01)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self._stop.set()
        self.thread.join(timeout=2)
        sm = [c for c, _ in self.rows]
        reasons = sorted({n for _, rs in self.rows for n in rs})
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": reasons, "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.mx, "reasons": reasons, "samples": len(sm),
                "source": "NVML every 10 ms during the timed region"}


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference algorithm; test infrastructure)
# ---------------------------------------------------------------------------


def _cpu_worker(conn, K, frames, seed, mode):
    from oracle import reference_port as rp
    from oracle import rng

    eng = rp.make_engine(mode, rp.Params(), rp.disk_offsets(5), direct=True)
    H, W = frames.shape[1:]
    s = eng.init(K, (W / 2.0, H / 2.0))
    stream = rng.LcgStream(seed)
    t = 0
    while True:
        msg = conn.recv()
        if msg is None:
            break
        nf = msg
        t0 = time.perf_counter()
        for _ in range(nf):
            eng.propagate(s, stream.normals(K))
            eng.likelihoods(s, frames[t % len(frames)])
            m = eng.max_loglik(s)
            tot = eng.weight_update(s, m)
            eng.normalize_and_scan(s, tot)
            eng.estimate(s)
            eng.resample(s, stream.uniform())
            t += 1
        conn.send(time.perf_counter() - t0)


class CpuArm:
    """P worker processes, each one independent track of the oracle port
    (restatement of halfpf's wide engine, filter.py:172-255, with the
    reference's direct (K, N) likelihood gather)."""

    def __init__(self, K, frames, mode, procs):
        import multiprocessing as mp

        ctx = mp.get_context("fork")
        self.procs = []
        for i in range(procs):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, args=(b, K, frames, 1000 + i, mode), daemon=True)
            p.start()
            self.procs.append((p, a))

    def step(self, frames_per_worker):
        t0 = time.perf_counter()
        for _, c in self.procs:
            c.send(frames_per_worker)
        for _, c in self.procs:
            c.recv()
        return time.perf_counter() - t0

    def close(self):
        for p, c in self.procs:
            try:
                c.send(None)
            except Exception:
                pass
            p.join(timeout=5)


def cpu_sample(cfg, mode="fp32", procs=1, frames=2, K=None):
    from oracle import reference_port as rp

    K = K or min(cfg["K"], 1_000_000)
    vid, _ = rp.generate_video(rp.Params(), max(frames, 2), cfg["W"], cfg["H"],
                               (cfg["W"] / 2.0, cfg["H"] / 2.0), 42)
    arm = CpuArm(K, vid, mode, procs)
    try:
        arm.step(1)  # warm (allocations, page faults)
        dt = arm.step(frames)
    finally:
        arm.close()
    return procs * K * frames / dt, dict(K=K, frames=frames, mode=mode, seconds=dt)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def run_reference_arm(args, cfg, rank, world):
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0))
    from oracle import reference_port as rp

    K = min(cfg["K"], 1_000_000)
    vid, _ = rp.generate_video(rp.Params(), 4, cfg["W"], cfg["H"], (cfg["W"] / 2.0, cfg["H"] / 2.0), 42)
    mode = "fp32" if cfg["precision"].startswith("fp16") else cfg["precision"]
    arm = CpuArm(K, vid, mode, procs)
    try:
        for _ in range(args.warmup):
            arm.step(1)
        times = [arm.step(1) for _ in range(args.steps)]
    finally:
        arm.close()
    tot = sum(times)
    value = procs * K * args.steps / tot
    sample = (f"oracle port of halfpf {mode} wide engine (oracle/reference_port.py: a NumPy restatement pinned "
              f"bit-exactly to halfpf, not halfpf itself -- /root/reference is absent on the GPU box; direct (K,81) "
              f"likelihood gather in chunks of 65536 particles, NumPy, 1 thread/process), "
              f"{procs} processes x 1 frame of {K} particles per step on {cfg['W']}x{cfg['H']}; "
              f"reference FP16 is pure-Python emulation, degenerate at K>=65536, so FP32 is the CPU arm")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_TAG[mode],
        "data": "synthetic", "config": _config_block(cfg, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_block(cfg, args):
    return {"workload": cfg["desc"], "width": cfg["W"], "height": cfg["H"], "frames": cfg["F"],
            "particles_per_track": cfg["K"], "tracks": cfg["tracks"], "precision": cfg["precision"],
            "tpb": args.tpb or "library default (fp16/fp32: 128 up to 2048 CTAs, else 256; fp64: 256)", "l2": "flushed (512 MiB write) before every timed step",
            "rng": "counter-based LCG (device)", "parallelism": f"tracks/GPU, {args.gpus} GPU(s), no collective"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

# ncu pipe names -> the microbenchmark kind that bounds them (pf_pipes.cu)
PIPE_PEAK_OF = {"fp16": "hfma2", "fma": "ffma", "fp64": "dfma", "alu": "lop3", "lsu": "lds", "xu": "mufu_ex2"}


def _ncu_profiles(config, prec):
    """Per-launch counters of the committed ncu captures (profiles/ncu_pipes.json:
    tools/pipes_capture.py; profiles/ncu_traffic.json: --set full)."""
    out = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        tr = d.get(f"{config}_{prec}") or d.get(f"{config}_{prec.split('-')[0]}")
        if tr:
            out["dram_bytes_per_launch"] = tr["dram_bytes_per_launch"]
            out["source"] = "profiles/ncu_traffic.json (ncu --set full)"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_pipes.json")) as fh:
            d = json.load(fh)
        out["pipes"] = d["configs"][config][prec]
    except Exception:
        pass
    return out


def pipe_block(ncu, live_ms, device, clk):
    """Per-pipe utilisation of the fused and map kernels: ncu per-launch
    warp-instruction counts per pipe / live launch time, against the per-pipe
    issue peaks measured on this box now (lib/libpf_pipes.so)."""
    if "pipes" not in ncu:
        return None
    try:
        import torch

        from paper_2308_00763_b200.pipes import pipe_peaks

        peaks = pipe_peaks(device)
    except Exception as e:  # noqa: BLE001
        return {"error": f"pipe microbenchmarks unavailable: {e}"}
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    mhz = (clk or {}).get("sm_mhz") or 1965
    out = {"peaks_warp_inst_per_sm_clk": peaks, "sm_mhz": mhz,
           "source": "counts: profiles/ncu_pipes.json (ncu sm__inst_executed_pipe_*); peaks: measured now"}
    for kern, ms in live_ms.items():
        c = ncu["pipes"].get(kern)
        if not c or not ms:
            continue
        if kern == "maps":
            ms = ms / max(1, c.get("launches_per_step", 1))
        cycles = ms * 1e-3 * mhz * 1e6 * sms  # SM-cycles of one launch
        row = {"ms_per_launch": ms}
        for pipe, pk in PIPE_PEAK_OF.items():
            if pipe in c:
                rate = c[pipe] / cycles
                row[pipe] = {"warp_inst_per_launch": c[pipe], "per_sm_clk": rate, "peak": peaks[pk],
                             "frac": rate / peaks[pk]}
        if "total" in c:
            row["issue"] = {"per_sm_clk": c["total"] / cycles, "peak": 4.0, "frac": c["total"] / cycles / 4.0,
                            "peak_source": "4 schedulers x 1 warp-instruction per clock"}
        out[kern] = row
    return out



def run_sharded(args, cfg, rank, world, local, dist, dev_frames, host_frames, truth, flush):
    """C5: one filter, particle range sharded over the ranks (strong scaling)."""
    import torch

    import paper_2308_00763_b200 as pf
    from paper_2308_00763_b200.sharded import DistShard
    from paper_2308_00763_b200.sharding import max_over_ranks

    F, K, W, H, prec = cfg["F"], cfg["K"], cfg["W"], cfg["H"], cfg["precision"]
    sh = DistShard(K, prec, W, H, 42, tpb=args.tpb or None, device=local)
    stream = sh.stream

    def steps(n, frames):
        tot = 0.0
        for _ in range(n):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            sh.reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            traj = sh.run(frames)
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot, traj

    steps(args.warmup, dev_frames)
    clocks = ClockSampler(local)
    clocks.start()
    dev_ms, traj = steps(args.steps, dev_frames)
    clk = clocks.stop()
    dev_ms = max_over_ranks(dev_ms, dist, device="cuda")
    value = K * F * args.steps / (dev_ms * 1e-3)
    rmse, mean_err, max_err = pf.accuracy_metrics(traj, truth)
    e2e_ms, _ = steps(args.steps, host_frames)  # frames H2D + trajectory D2H inside the events
    e2e_s = max_over_ranks(e2e_ms, dist, device="cuda") * 1e-3
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPE_TAG[prec], "data": "synthetic",
            "config": dict(_config_block(cfg, args), parallelism=(
                f"one filter, particle range over {world} GPUs: 3 all-gathers (8 B, 32 B, 4 B per rank) "
                f"per frame on the library stream (NCCL), remote ancestors read over CUDA-IPC peer mappings")),
            "e2e": {"value": K * F * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(host_frames.nbytes),
                    "d2h_bytes_per_step": int(F * 2 * 8),
                    "timer": "CUDA events on the library stream around run(host frames), max over ranks"},
            "roofline": None, "cpu_baseline": None, "clocks": clk,
            "gpu_launches": (4 * F + 1) * args.steps,
            "tracking": {"rmse_px": rmse, "mean_err_px": mean_err, "max_err_px": max_err},
        }
        print(json.dumps(line), flush=True)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()



def relaunch(n: int) -> None:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        raise SystemExit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default=None)
    ap.add_argument("--tpb", type=int, default=0, help="threads per block (0 = library default per precision)")
    ap.add_argument("--particles", type=int, default=0,
                    help="override particles per track (e.g. one shard's share of C5: 2^30 / N)")
    ap.add_argument("--tracks", type=int, default=0,
                    help="override the config's track count (e.g. one rank's share of C4: 8192 / N)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the FP32/FP64 side measurements")
    ap.add_argument("--profile-only", action="store_true", help="(ncu) run 1 untimed step, no JSON")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.precision:
        cfg["precision"] = args.precision
    if args.tracks:
        cfg["tracks"] = args.tracks
    if args.particles:
        cfg["K"] = args.particles
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: re-run this command
        # under torchrun, one rank per GPU (127.0.0.1 rendezvous)
        relaunch(args.gpus)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (one rank per GPU)")
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return

    import torch

    # PF_BENCH_SHARE_GPU=1 (test hook): more ranks than GPUs -- ranks share
    # devices round-robin and synchronise over gloo (NCCL needs one GPU per
    # rank); exercises the N-rank path on a one-GPU box.  Not a measurement.
    share = os.environ.get("PF_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2308_00763_b200 as pf

    from paper_2308_00763_b200.sharding import max_over_ranks, shard_tracks

    # batched independent tracks, block-partitioned over ranks (C2 at N GPUs:
    # one independent track per rank); global track g -> seed 42+g, video g % nv
    total_tracks = cfg["tracks"] if cfg["tracks"] > 1 else world
    shard = shard_tracks(total_tracks, world, rank)
    tracks = shard.count
    F, K, W, H = cfg["F"], cfg["K"], cfg["W"], cfg["H"]
    nv = cfg["videos"]
    vids, truths = [], []
    for j in range(nv):
        v = pf.generate_video(pf.ModelParams(), F, W, H, (W / 2.0, H / 2.0), 42 + j)
        vids.append(v.frames)
        truths.append(v.truth)
    rot = shard.first % nv  # local track i observes video (first + i) % nv
    vids = vids[rot:] + vids[:rot]
    truths = truths[rot:] + truths[:rot]
    # e2e inputs come from pinned host memory (the contract's H2D leg): a page-
    # locked buffer the copy engine reads directly
    pinned = torch.from_numpy(np.ascontiguousarray(np.stack(vids)) if nv > 1 else vids[0]).pin_memory()
    host_frames = pinned.numpy()
    dev_frames = pinned.cuda()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    seeds = shard.seeds(42)

    def make(precision):
        return pf.Filter(K, precision, W, H, seeds=seeds, n_tracks=tracks, n_videos=nv, tpb=args.tpb,
                         device=local)

    def device_steps(f, n, timed=True, parts=None):
        tot = 0.0
        launches = 0
        for _ in range(n):
            flush.zero_()
            torch.cuda.synchronize()
            f.reset()
            f.run_frames(dev_frames, F)
            tm = f.timings()
            tot += tm["total"]
            launches += f.launches()
            if parts is not None:
                parts.append(tm)
        return tot, launches

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def over_ranks(x):
        return max_over_ranks(x, dist, device="cuda")

    prec = cfg["precision"]
    if cfg.get("sharded") and world > 1:
        run_sharded(args, cfg, rank, world, local, dist, dev_frames, host_frames, truths[0], flush)
        return
    f = make(prec)
    if args.profile_only:
        f.run_frames(dev_frames, F)
        torch.cuda.synchronize()
        return
    device_steps(f, args.warmup)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    parts = []
    dev_ms, launches = device_steps(f, args.steps, parts=parts)
    barrier()
    clk = clocks.stop()
    dev_ms = over_ranks(dev_ms)
    updates_per_step = total_tracks * K * F
    value = updates_per_step * args.steps / (dev_ms * 1e-3)
    f.reset()
    traj = f.run_frames(dev_frames, F)
    truth = truths[0]
    rmse, mean_err, max_err = pf.accuracy_metrics(traj[0], truth)

    # ---- e2e through the host-buffer C-ABI call (H2D + D2H inside) --------
    f.reset()
    f.run_frames(host_frames, F)  # untimed: the host path's first call sizes its frame buffer
    barrier()
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        f.reset()
        t0 = time.perf_counter()
        f.run_frames(host_frames, F)
        e2e_s += time.perf_counter() - t0
    barrier()
    e2e_s = over_ranks(e2e_s)
    e2e = {"value": updates_per_step * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(host_frames.nbytes), "d2h_bytes_per_step": int(tracks * F * 2 * 8),
           "ms_per_step": 1e3 * e2e_s / args.steps, "timer": "wall clock around pf_run (pinned host frames)"}

    # ---- roofline of the dominant kernel (fused frame kernel) ------------
    # Timed inside the production schedule: the per-frame launch pair (fused
    # kernel + its tile table, programmatic dependent launch, replayed from a
    # CUDA graph) of the timed steps above -- device time of the frame region
    # (CUDA events on the library stream around the graph) / F.  The pair
    # overlaps under PDL, so this per-launch time is the frame period; the
    # serialised per-kernel split (events between launches, no graph) gives
    # the fused kernel's share of it.
    frames_ms = statistics.mean(t["frames"] for t in parts)
    maps_ms = statistics.mean(t["maps"] for t in parts)
    period_ms = frames_ms / F
    f.set_profiling(True)
    flush.zero_()
    torch.cuda.synchronize()
    f.reset()
    f.run_frames(dev_frames, F)
    tm = f.timings()
    f.set_profiling(False)
    s = SIZES[prec]
    share = tm["frames"] / (tm["frames"] + tm["tables"])
    bytes_per_launch = tracks * K * 6 * s + nv * W * H
    peak, peak_src = _peaks()
    achieved = bytes_per_launch / (period_ms * 1e-3) / 1e9
    ncu = _ncu_profiles(args.config, prec)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu.get("dram_bytes_per_launch"), "kernel": f"pf_fused_frame<{prec}>",
                "algorithmic_bytes_per_launch": bytes_per_launch, "bytes_per_particle": 6 * s,
                "avg_launch_ms": period_ms,
                "timing": ("in the production schedule: frame-region device time of the timed steps / F "
                           "(fused + tile table per frame, PDL-overlapped, CUDA graph)"),
                "frames_x_launch_ms": frames_ms, "ms_per_step": dev_ms / args.steps,
                "serialised": {"fused_ms": tm["frames"] / F, "tile_table_ms": tm["tables"] / F,
                               "fused_share": share,
                               "how": "events between launches, no graph, no PDL overlap (one extra step)"},
                "maps_ms_per_step": maps_ms, "peak_source": peak_src,
                "traffic_source": ncu.get("source")}
    assert frames_ms <= dev_ms / args.steps * (1 + 1e-6), (frames_ms, dev_ms / args.steps)
    pipes_line = pipe_block(ncu, {"fused": period_ms, "maps": maps_ms}, local, clk)
    if pipes_line:
        roofline["pipes"] = pipes_line
    f.close()

    # ---- the other precisions of the same workload -----------------------
    extra = {}
    if not args.no_extra and args.config == "c2":
        for p2 in ("fp16", "fp32", "fp64"):
            g = make(p2)
            device_steps(g, 2)
            parts2 = []
            ms2, _ = device_steps(g, max(3, args.steps // 2), parts=parts2)
            ms2 = over_ranks(ms2)
            v2 = updates_per_step * max(3, args.steps // 2) / (ms2 * 1e-3)
            g.reset()
            t2 = g.run_frames(dev_frames, F)
            e2 = pf.accuracy_metrics(t2[0], truth)
            per2 = statistics.mean(t["frames"] for t in parts2) / F
            b2 = tracks * K * 6 * SIZES[p2] + nv * W * H
            extra[p2] = {"value": v2, "unit": UNIT, "tracking_rmse_px": e2[0], "tracking_mean_err_px": e2[1],
                         "frame_period_ms": per2, "hbm_frac": b2 / (per2 * 1e-3) / 1e9 / peak}
            pl = pipe_block(_ncu_profiles(args.config, p2),
                            {"fused": per2, "maps": statistics.mean(t["maps"] for t in parts2)}, local, clk)
            if pl:
                extra[p2]["pipes"] = pl
            g.close()
        extra[prec] = {"value": value, "unit": UNIT, "tracking_rmse_px": rmse, "tracking_mean_err_px": mean_err,
                       "frame_period_ms": period_ms, "hbm_frac": achieved / peak}
        extra["fp16_over_fp32"] = value / extra["fp32"]["value"]
        extra["fp16_over_fp64"] = value / extra["fp64"]["value"]
        extra["packed_over_scalar_fp16"] = value / extra["fp16"]["value"]

    # ---- per-frame API latency: Filter.step (the reference's per-frame run
    # and estimate, filter.py:617-654) on host frames and on device frames
    step_lat = None
    if not args.no_extra and tracks == 1:
        g = make(prec)
        host1 = np.ascontiguousarray(host_frames[:F] if nv == 1 else host_frames[0])
        lat = {}
        for label, src in (("host_frame", host1), ("device_frame", dev_frames if nv == 1 else dev_frames[0])):
            g.reset()
            for t in range(5):
                g.step(src[t])
            g.reset()
            n_lat = min(F, 50)
            t0 = time.perf_counter()
            for t in range(n_lat):
                g.step(src[t])
            lat[label] = {"us_per_frame": 1e6 * (time.perf_counter() - t0) / n_lat, "frames": n_lat}
        g.close()
        step_lat = dict(lat, api="Filter.step(frame) -> (x, y): frame in, likelihood map, fused frame kernel, "
                                 "tile table (estimate written to host-mapped memory), host sync -- wall clock per call",
                        particles=K, precision=prec)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mode = "fp32" if prec.startswith("fp16") else prec
        rate, info = cpu_sample(cfg, mode=mode, procs=1, frames=2)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": (f"oracle port of halfpf {mode} wide engine (oracle/reference_port.py, a restatement pinned "
                          f"to halfpf; direct (K,81) gather chunked at 65536), {info['frames']} frames "
                          f"of {info['K']} particles on the C2 video ({info['seconds']:.1f} s); reference FP16 is "
                          f"pure-Python emulation and degenerate at K>=65536"),
               "cpu": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            # a fixed batch of tracks split over the ranks is strong scaling; one
            # independent track per rank (C2 at N GPUs) is weak scaling
            "scaling": "strong" if cfg["tracks"] > 1 else "weak", "vs_baseline": None,
            "dtype": DTYPE_TAG[prec], "data": "synthetic",
            "config": _config_block(cfg, args),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
            "gpu_launches": launches,
            "tracking": {"rmse_px": rmse, "mean_err_px": mean_err, "max_err_px": max_err},
            "by_precision": extra or None,
            "step_latency": step_lat,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
