"""The ctypes stub of INTEGRATION.md §2 -- what a `halfpf` maintainer would
paste next to filter.run -- executed as written against the built library:
it must return the same trajectory as this package's `run()`."""

import os
import re
import types

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _stub_source():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## 2."):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    lib = os.path.join(ROOT, "paper_2308_00763_b200", "lib", "libpf_b200.so")
    return code.replace('C.CDLL("libpf_b200.so")', f"C.CDLL({lib!r})")


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16-packed"])
def test_integration_stub_matches_package(mode):
    import paper_2308_00763_b200 as pf

    ns = {"DegeneracyError": pf.DegeneracyError}
    exec(compile(_stub_source(), "INTEGRATION.md#2", "exec"), ns)
    video = pf.generate_video(pf.ModelParams(), 12, 96, 80, (40.0, 30.0), 3)
    p = pf.ModelParams()
    tmpl = pf.disk_template(p.disk_radius)
    got = ns["run_b200"](video, 20_000, types.SimpleNamespace(value=mode), 7, p, tmpl, (48.0, 40.0))
    ref = pf.run(video, 20_000, mode, 7, start_hint=(48.0, 40.0)).trajectory
    assert np.array_equal(got, ref)
