"""C-ABI surface (CPU): the library loads and exports every declared symbol;
host-built tables match the oracle.  No device compute here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "pf_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_reference_entry_points():
    names = _declared()
    for must in ("pf_create", "pf_run", "pf_step", "pf_destroy", "pf_stage_propagate", "pf_stage_likelihood",
                 "pf_stage_max", "pf_stage_weight", "pf_stage_normalize", "pf_stage_estimate",
                 "pf_stage_resample", "pf_systematic_ancestors", "pf_rng_normals"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2308_00763_b200 import _native as N

    L = N.lib()
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    bound = {s[0] for s in N.SIGNATURES}
    assert set(_declared()) == bound
    assert b"sm_100a" in L.pf_version()


def test_library_built_for_sm100a():
    from paper_2308_00763_b200 import _native as N

    blob = open(N.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_exp16_table_matches_oracle():
    from oracle import reference_port as rp
    from paper_2308_00763_b200 import _native as N

    out = np.empty(65536, dtype=np.uint16)
    assert N.lib().pf_exp16_table(N.ptr(out)) == 0
    ref = rp.exp16_table().view(np.uint16)
    nan = np.isnan(rp.exp16_table().astype(np.float32))
    assert np.array_equal(out[~nan], ref[~nan])
    assert np.all(np.isnan(out[nan].view(np.float16)))


def test_python_api_validation_mirrors_reference():
    from paper_2308_00763_b200 import filter as F

    with pytest.raises(ValueError, match="unknown precision"):
        F.PrecisionMode.from_name("fp8")
    with pytest.raises(ValueError, match="at least 2"):
        F._validate_k(1, F.PrecisionMode.FP64)
    with pytest.raises(ValueError, match="even"):
        F._validate_k(3, F.PrecisionMode.FP16_PACKED)
    F._validate_k(1 << 24, F.PrecisionMode.FP16_PACKED)


def test_pipes_library_exports_declared_symbols():
    from paper_2308_00763_b200 import pipes

    src = open(os.path.join(ROOT, "include", "pf_pipes.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", src))
    L = pipes.lib()
    assert all(hasattr(L, n) for n in names)
    assert names == {s[0] for s in pipes.SIGNATURES}
    assert L.pf_pipe_count() == 12 and L.pf_pipe_name(0) == b"hfma2"
