"""Input side of the step: device video rendering and PFVD
ingest.  The device renderer equals its restatement (oracle/video.py: the
reference model with the LCG noise stream) byte-for-byte and reproduces the
reference trajectory exactly; the PFVD reader returns the written pixels and
the reference's error messages."""

import numpy as np
import pytest

from oracle import reference_port as rp
from oracle import video as ov

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("F,W,H,start,seed", [(5, 128, 128, (64.0, 64.0), 42), (7, 61, 37, (2.0, 35.5), 9),
                                               (3, 1024, 1024, (512.0, 512.0), 1)])
def test_device_video_matches_oracle(F, W, H, start, seed):
    import paper_2308_00763_b200 as pf

    frames, truth = pf.generate_video_device(pf.ModelParams(), F, W, H, start, seed)
    ref, rtruth = ov.generate_video_lcg(rp.Params(), F, W, H, start, seed)
    assert np.array_equal(frames.cpu().numpy(), ref)
    assert np.array_equal(truth, rtruth)
    # same trajectory as the reference (NumPy) generator
    host = pf.generate_video(pf.ModelParams(), F, W, H, start, seed)
    assert np.array_equal(truth, host.truth)


def test_device_video_statistics_match_reference_model():
    import paper_2308_00763_b200 as pf

    dev, truth = pf.generate_video_device(pf.ModelParams(), 20, 128, 128, (64.0, 64.0), 3)
    host = pf.generate_video(pf.ModelParams(), 20, 128, 128, (64.0, 64.0), 3)
    a = dev.cpu().numpy().astype(np.float64)
    b = host.frames.astype(np.float64)
    # background mean/std and disk contrast agree with the NumPy renderer
    assert abs(a.mean() - b.mean()) < 0.05
    assert abs(a.std() - b.std()) < 0.05
    assert np.array_equal(a > 164, b > 164)  # noise 5 px never crosses the bg/fg midpoint


def test_device_video_tracks(tmp_path):
    import paper_2308_00763_b200 as pf

    frames, truth = pf.generate_video_device(pf.ModelParams(), 30, 128, 128, (64.0, 64.0), 5)
    traj = pf.Filter(100_000, "fp16", 128, 128, 42).run(frames)
    err = np.mean(np.hypot(*(traj - truth).T))
    assert err < 1.0


def test_pfvd_device_reader(tmp_path):
    import paper_2308_00763_b200 as pf

    v = pf.generate_video(pf.ModelParams(), 9, 77, 41, (30.0, 20.0), 4)
    path = tmp_path / "v.pfvd"
    pf.write_video(path, v)
    got = pf.read_video_device(path)
    assert got.shape == (9, 41, 77)
    assert np.array_equal(got.cpu().numpy(), v.frames)
    # large file: several staging chunks
    big = pf.Video(frames=np.random.default_rng(0).integers(0, 256, (40, 512, 512), dtype=np.uint8),
                   truth=np.zeros((40, 2)))
    pf.write_video(tmp_path / "b.pfvd", big)
    assert np.array_equal(pf.read_video_device(tmp_path / "b.pfvd").cpu().numpy(), big.frames)


def test_pfvd_errors_match_reference(tmp_path):
    import paper_2308_00763_b200 as pf

    bad = tmp_path / "bad.pfvd"
    bad.write_bytes(b"XXXX" + b"\0" * 12)
    with pytest.raises(ValueError, match="bad container magic at offset 0"):
        pf.read_video_device(bad)
    short = tmp_path / "short.pfvd"
    short.write_bytes(b"PFVD\x01\0")
    with pytest.raises(ValueError, match="truncated header at offset 4"):
        pf.read_video_device(short)
    trunc = tmp_path / "trunc.pfvd"
    trunc.write_bytes(b"PFVD" + np.array([2, 4, 4], dtype="<u4").tobytes() + b"\0" * 20)
    with pytest.raises(ValueError, match="expected 32 pixel bytes at offset 16, got 20"):
        pf.read_video_device(trunc)
    with pytest.raises(FileNotFoundError):
        pf.read_video_device(tmp_path / "missing.pfvd")
