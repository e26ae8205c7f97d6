"""B200-native particle-filter tracking step (arXiv 2308.00763), drop-in for `halfpf`.

Public names mirror /root/reference/pkg/src/halfpf/__init__.py:3-33.  Every
tracking computation runs in the sm_100a library lib/libpf_b200.so (C ABI in
include/pf_b200.h); importing the filter API without it raises.
"""

from .model import (
    ModelParams,
    PixelTemplate,
    Video,
    disk_template,
    generate_video,
    generate_video_device,
    read_truth_csv,
    read_video_device,
    read_video,
    write_truth_csv,
    write_video,
)
from .filter import (
    MAX_PARTICLES,
    STAGES,
    DegeneracyError,
    Filter,
    OpCounters,
    ParticleSet,
    PhiloxRngStream,
    PrecisionMode,
    RngStream,
    RunResult,
    accuracy_metrics,
    init_particles,
    make_engine,
    run,
    systematic_ancestors,
)

__all__ = [
    "ModelParams", "PixelTemplate", "Video", "disk_template", "generate_video", "generate_video_device",
    "read_video_device",
    "read_video", "write_video", "read_truth_csv", "write_truth_csv",
    "MAX_PARTICLES", "STAGES", "DegeneracyError", "Filter", "OpCounters", "ParticleSet",
    "PhiloxRngStream", "PrecisionMode", "RngStream", "RunResult", "accuracy_metrics", "init_particles",
    "make_engine", "run", "systematic_ancestors",
]
