"""GPU parity of the per-frame likelihood maps (filter.py:204-217 wide,
384-423 binary16): every map entry equals the oracle's reference-formula
likelihood at that clamped rint position, bit-for-bit -- for the disk
template, other radii, an asymmetric custom template, odd frame shapes and
the 1024x1024 C3 frame in every mode, and a template over 128 offsets
(several NumPy pairwise leaves: the generic plan kernel)."""

import numpy as np
import pytest

from oracle import reference_port as rp

pytestmark = pytest.mark.gpu


def _maps(mode, frames, template=None, params=None):
    import paper_2308_00763_b200 as pf

    F, H, W = frames.shape
    f = pf.Filter(64, mode, W, H, 1, template=template, params=params)
    out = f.likelihood_maps(frames)
    f.close()
    return out


def _oracle(mode, frame, offs, p):
    if mode.startswith("fp16"):
        return rp.loglik_map_half(frame, offs, p)
    return rp.loglik_map_wide(frame, offs, p, np.float64 if mode == "fp64" else np.float32)


@pytest.mark.parametrize("mode", ["fp16", "fp16-packed", "fp32", "fp64"])
@pytest.mark.parametrize("W,H", [(128, 128), (77, 53), (96, 80)])
def test_maps_disk_template(mode, W, H):
    frames, _ = rp.generate_video(rp.Params(), 3, W, H, (W / 2.0, H / 2.0), 7)
    got = _maps(mode, frames)
    offs = rp.disk_offsets(5)
    for t in range(3):
        ref = _oracle(mode, frames[t], offs, rp.Params())
        half = mode.startswith("fp16")
        assert np.array_equal(got[t].view(np.uint16 if half else got.dtype).ravel(),
                              ref.astype(got.dtype).view(np.uint16 if half else got.dtype).ravel())


@pytest.mark.parametrize("mode", ["fp16", "fp16-packed"])
def test_maps_c3_frame_fp16(mode):
    frames, _ = rp.generate_video(rp.Params(), 1, 1024, 1024, (512.0, 512.0), 42)
    got = _maps(mode, frames)[0]
    ref = _oracle(mode, frames[0], rp.disk_offsets(5), rp.Params())
    assert np.array_equal(got.view(np.uint16), ref.view(np.uint16))


@pytest.mark.parametrize("mode", ["fp16", "fp64"])
def test_maps_other_templates(mode):
    import paper_2308_00763_b200 as pf

    frames, _ = rp.generate_video(rp.Params(), 2, 61, 47, (30.0, 20.0), 3)
    # radius 3 disk
    t3 = pf.disk_template(3)
    got = _maps(mode, frames, template=t3, params=pf.ModelParams(disk_radius=3))
    ref = _oracle(mode, frames[1], rp.disk_offsets(3), rp.Params(disk_radius=3))
    assert np.array_equal(np.asarray(got[1], dtype=np.float64), np.asarray(ref, dtype=np.float64))
    # asymmetric custom template (odd tap parities, negative and positive offsets)
    offs = np.array([[0, 0], [3, -2], [-1, 4], [2, 2], [-4, -1], [1, 0]], dtype=np.int64)
    tmpl = pf.PixelTemplate(offs)
    got = _maps(mode, frames, template=tmpl)
    ref = _oracle(mode, frames[0], offs, rp.Params())
    assert np.array_equal(np.asarray(got[0], dtype=np.float64), np.asarray(ref, dtype=np.float64))


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
def test_maps_c3_frame_wide(mode):
    # 1024-wide frames: 8-row bands, FP64 on 1024-thread CTAs (pf_map_wide_img)
    frames, _ = rp.generate_video(rp.Params(), 1, 1024, 1024, (512.0, 512.0), 42)
    got = _maps(mode, frames)[0]
    ref = _oracle(mode, frames[0], rp.disk_offsets(5), rp.Params())
    assert np.array_equal(got, ref.astype(got.dtype))


@pytest.mark.parametrize("mode", ["fp16", "fp32", "fp64"])
def test_maps_template_over_128_offsets(mode):
    # > 128 offsets: NumPy's pairwise sum splits into several leaves (generic
    # pf_map_wide plan evaluation for FP32 / FP64)
    import paper_2308_00763_b200 as pf

    frames, _ = rp.generate_video(rp.Params(disk_radius=7), 2, 70, 58, (35.0, 29.0), 5)
    offs = rp.disk_offsets(7)
    assert len(offs) > 128
    got = _maps(mode, frames, template=pf.disk_template(7), params=pf.ModelParams(disk_radius=7))
    for t in range(2):
        ref = _oracle(mode, frames[t], offs, rp.Params(disk_radius=7))
        assert np.array_equal(np.asarray(got[t], dtype=np.float64), np.asarray(ref, dtype=np.float64))


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
@pytest.mark.parametrize("bg,fg,scale", [(100.0, 228.0, 37.5), (99.5, 230.25, 50.0), (-3.0, 1000.0, 50.0)])
def test_maps_params_integer_and_fractional_means(mode, bg, fg, scale):
    # integral means within the exactness bound: integer row-prefix kernel;
    # fractional means (or terms too large): the term-image kernel
    import paper_2308_00763_b200 as pf

    frames, _ = rp.generate_video(rp.Params(), 2, 83, 41, (40.0, 20.0), 9)
    got = _maps(mode, frames, params=pf.ModelParams(bg_mean=bg, fg_mean=fg, likelihood_scale=scale))
    for t in range(2):
        ref = _oracle(mode, frames[t], rp.disk_offsets(5), rp.Params(bg_mean=bg, fg_mean=fg, likelihood_scale=scale))
        assert np.array_equal(got[t], ref.astype(got.dtype))


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
def test_maps_duplicate_offsets(mode):
    # a template with a repeated offset is a multiset, not a union of runs
    import paper_2308_00763_b200 as pf

    frames, _ = rp.generate_video(rp.Params(), 1, 64, 48, (30.0, 20.0), 4)
    offs = np.array([[0, 0], [1, 0], [1, 0], [2, 0], [-1, 2], [0, 2]], dtype=np.int64)
    got = _maps(mode, frames, template=pf.PixelTemplate(offs))
    ref = _oracle(mode, frames[0], offs, rp.Params())
    assert np.array_equal(got[0], ref.astype(got.dtype))
