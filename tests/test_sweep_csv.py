"""Sweep harness / CSV schema (halfpf.bench, bench.py:20-190): same header,
same row format as the reference module for identical records (CPU), and a
small device sweep end to end (GPU)."""

import math
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, have_reference


def _records(mod, PM):
    recs = [
        mod.BenchRecord(mode=PM.FP16_SCALAR, K=4096, workers=128, repeat_index=1, total_ms=12.5,
                        per_stage_ms={"propagate": 3.25, "likelihood": 0.5, "max": 0.0, "weight": 0.0,
                                      "normalize": 0.0, "resample": 0.0},
                        rmse_vs_truth=0.75, mean_err_vs_fp64=0.0625),
        mod.BenchRecord(mode=PM.FP64, K=10, workers=1, repeat_index=0, error="particle count"),
        mod.BenchRecord(mode=PM.FP32, K=64, workers=2, repeat_index=3, total_ms=1.0, per_stage_ms={},
                        rmse_vs_truth=math.inf, mean_err_vs_fp64=0.1, timings_reliable=False),
    ]
    return recs


def test_csv_header_and_rows(tmp_path):
    from paper_2308_00763_b200 import PrecisionMode
    from paper_2308_00763_b200 import bench as sweep

    assert sweep.CSV_HEADER.split(",")[:4] == ["mode", "K", "workers", "repeat"]
    recs = _records(sweep, PrecisionMode)
    p = tmp_path / "b.csv"
    sweep.write_csv(recs, p)
    rows = sweep.read_csv(p)
    assert [r["mode"] for r in rows] == ["fp16", "fp64", "fp32"]
    assert rows[0]["t_propagate"] == "3.25" and rows[1]["total_ms"] == "nan" and rows[2]["total_ms"] == "nan"
    assert rows[2]["rmse"] == "nan"
    assert sweep.tpb_for_workers(256) == 256 and sweep.tpb_for_workers(4) is None


@pytest.mark.skipif(not have_reference(), reason="reference sources not present")
def test_rows_identical_to_reference_module():
    sys.path.insert(0, REFERENCE_SRC)
    try:
        from halfpf import bench as ref
        from halfpf.filter import PrecisionMode as RPM
    finally:
        sys.path.remove(REFERENCE_SRC)
    from paper_2308_00763_b200 import PrecisionMode
    from paper_2308_00763_b200 import bench as sweep

    assert sweep.CSV_HEADER == ref.CSV_HEADER
    for a, b in zip(_records(sweep, PrecisionMode), _records(ref, RPM)):
        assert sweep.record_to_row(a) == ref.record_to_row(b)


@pytest.mark.gpu
def test_device_sweep_end_to_end(tmp_path):
    import paper_2308_00763_b200 as pf
    from paper_2308_00763_b200 import bench as sweep

    video = pf.generate_video(pf.ModelParams(), 12, 96, 96, (48.0, 48.0), 5)
    modes = [pf.PrecisionMode.FP64, pf.PrecisionMode.FP32, pf.PrecisionMode.FP16_SCALAR, pf.PrecisionMode.FP16_PACKED]
    recs = sweep.run_sweep(video, [1, 4096, 30000], modes, [1, 128, 1024], 2, 7)
    assert len(recs) == 4 * 3 * 3 * 2
    bad = [r for r in recs if r.error is not None]
    assert bad and all(r.K == 1 for r in bad)  # K < 2 becomes an error row, not a crash
    good = [r for r in recs if r.error is None]
    for r in good:
        assert r.total_ms > 0 and math.isfinite(r.rmse_vs_truth)
        if r.mode == pf.PrecisionMode.FP64:
            assert r.mean_err_vs_fp64 == 0.0
        if r.mode == pf.PrecisionMode.FP32 and r.K == 30000:
            assert r.mean_err_vs_fp64 < 0.5
    # TPB never changes a trajectory: same (mode, K, repeat) -> same accuracy columns
    key = {}
    for r in good:
        key.setdefault((r.mode, r.K, r.repeat_index), set()).add((r.rmse_vs_truth, r.mean_err_vs_fp64))
    assert all(len(v) == 1 for v in key.values())
    p = tmp_path / "sweep.csv"
    sweep.write_csv(recs, p)
    assert len(sweep.read_csv(p)) == len(recs)
