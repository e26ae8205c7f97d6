"""Benchmark sweep harness over the device filter (mirrors halfpf.bench).

Reference: /root/reference/pkg/src/halfpf/bench.py:20-190 -- precision x
particle-count x worker-count sweeps, per-stage timings, accuracy against the
ground truth and drift against an FP64 run of the same draws, serialised to a
fixed-schema CSV that pfreport reads.  Same names, fields, CSV header and row
format here; what changes is what the columns measure:

  * every configuration runs the fused device path (`filter.run`);
  * `workers` is the paper's threads-per-block sweep: a value in
    {32, 64, 128, 256, 512, 1024} selects that TPB, any other value (the
    reference's 1/2/4/8 thread-pool sizes) runs the library default TPB and is
    recorded as given (results never depend on TPB -- DESIGN.md);
  * stage times are device-event times mapped onto the reference's keys: the
    likelihood-map build is `t_likelihood`, the fused per-frame kernels are
    `t_propagate` (fused kernels report against their first stage), the other
    stage columns are 0; `total_ms` is the wall time of the run;
  * the op-counter columns are 0 (ncu pipe metrics replace them).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .filter import STAGES, DegeneracyError, PrecisionMode, accuracy_metrics, run
from .model import ModelParams, PixelTemplate, Video

CSV_HEADER = (
    "mode,K,workers,repeat,total_ms,t_propagate,t_likelihood,t_max,"
    "t_weight,t_normalize,t_resample,rmse,mean_err_fp64,widen,narrow,"
    "half_arith,wide_arith,special_fn"
)

TPB_VALUES = (32, 64, 128, 256, 512, 1024)


@dataclass
class BenchRecord:
    mode: PrecisionMode
    K: int
    workers: int
    repeat_index: int
    total_ms: float = math.nan
    per_stage_ms: Dict[str, float] = field(default_factory=dict)
    rmse_vs_truth: float = math.nan
    mean_err_vs_fp64: float = math.nan
    widen_count: int = 0
    narrow_count: int = 0
    half_arith_count: int = 0
    wide_arith_count: int = 0
    special_fn_count: int = 0
    timings_reliable: bool = True
    error: Optional[str] = None


def _derived_seed(seed: int, repeat: int) -> int:
    return int(seed) + repeat  # bench.py:64-65


def tpb_for_workers(workers: int) -> Optional[int]:
    return int(workers) if int(workers) in TPB_VALUES else None


def run_sweep(
    video: Video,
    Ks: Sequence[int],
    modes: Sequence[PrecisionMode],
    workers_list: Sequence[int],
    repeats: int,
    seed: int,
    params: Optional[ModelParams] = None,
    template: Optional[PixelTemplate] = None,
    start_hint: Optional[Tuple[float, float]] = None,
    concurrent_configs: bool = False,
    device: int = 0,
) -> List[BenchRecord]:
    """Run every configuration; failures become rows, not crashes (bench.py:68-149)."""
    fp64_cache: Dict[Tuple[int, int], np.ndarray] = {}

    def fp64_reference(K: int, run_seed: int) -> np.ndarray:
        key = (K, run_seed)
        if key not in fp64_cache:
            fp64_cache[key] = run(video, K, PrecisionMode.FP64, run_seed, params=params, template=template,
                                  start_hint=start_hint, device=device).trajectory
        return fp64_cache[key]

    configs = [(K, mode, workers, repeat) for K in Ks for mode in modes for workers in workers_list
               for repeat in range(repeats)]

    def execute(config) -> BenchRecord:
        K, mode, workers, repeat = config
        record = BenchRecord(mode=mode, K=K, workers=workers, repeat_index=repeat)
        run_seed = _derived_seed(seed, repeat)
        try:
            result = run(video, K, mode, run_seed, workers=workers, params=params, template=template,
                         start_hint=start_hint, tpb=tpb_for_workers(workers), device=device)
        except (ValueError, DegeneracyError) as err:
            record.error = str(err)
            return record
        record.total_ms = result.total_ms
        record.per_stage_ms = dict(result.stage_ms)
        # tracked positions are whole pixels; round estimates before scoring (bench.py:127-130)
        record.rmse_vs_truth = accuracy_metrics(np.rint(result.trajectory), video.truth)[0]
        record.mean_err_vs_fp64 = accuracy_metrics(result.trajectory, fp64_reference(K, run_seed))[1]
        record.timings_reliable = not concurrent_configs
        return record

    if concurrent_configs:
        with ThreadPoolExecutor() as pool:
            return list(pool.map(execute, configs))
    return [execute(cfg) for cfg in configs]


def _fmt(value: float) -> str:
    return "nan" if not math.isfinite(value) else repr(float(value))


def record_to_row(record: BenchRecord) -> str:
    """bench.py:156-183, same field order and formatting."""
    if record.error is not None:
        times = ["nan"] * 7
        metrics = ["nan", "nan"]
    else:
        stage = record.per_stage_ms
        if record.timings_reliable:
            times = [_fmt(record.total_ms)] + [_fmt(stage.get(name, math.nan)) for name in STAGES]
        else:
            times = ["nan"] * 7
        metrics = [_fmt(record.rmse_vs_truth), _fmt(record.mean_err_vs_fp64)]
    fields = ([record.mode.value, str(record.K), str(record.workers), str(record.repeat_index)] + times + metrics +
              [str(record.widen_count), str(record.narrow_count), str(record.half_arith_count),
               str(record.wide_arith_count), str(record.special_fn_count)])
    return ",".join(fields)


def write_csv(records: Sequence[BenchRecord], path) -> None:
    with open(path, "w", newline="") as fh:
        fh.write(CSV_HEADER + "\n")
        for record in records:
            fh.write(record_to_row(record) + "\n")


def read_csv(path) -> List[Dict[str, str]]:
    """Rows of a sweep CSV as dicts (header checked)."""
    with open(path) as fh:
        header = fh.readline().strip()
        if header != CSV_HEADER:
            raise ValueError(f"{path}: unexpected header {header!r}")
        keys = header.split(",")
        return [dict(zip(keys, line.strip().split(","))) for line in fh if line.strip()]
