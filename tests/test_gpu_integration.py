"""GPU: the reference's own caller code (tests/cpp/ref_dropin.cpp, compiled against the
UNMODIFIED reference headers by oracle/Makefile) with fwa::backbone::run_backbone
swapped for fwa::b200::run_backbone (include/fwa_b200.hpp): integer outputs equal,
features within the bf16 tolerance, error taxonomy preserved."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ref_dropin not built (needs /root/reference)")
def test_reference_caller_drop_in():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert out["ints_equal"] and out["numeric_error"]
    assert out["rel_err"] <= 1e-2
    assert out["stream_equal"]  # Backbone::run_frames == run per frame, bit for bit
    assert out["empty_numeric_error"]  # empty PillarSet -> numeric_error, as backbone.hpp:218-222
    assert out["stages_ok"], out["stages_ms"]  # RunStats.stages filled (bench_group reads them)
    assert out["proj_ok"] and out["proj_rel_err"] <= 1e-2  # BackboneParams::input_proj on the device
    assert out["proj_width_shape_error"]
    assert out["concurrent_ok"]  # two threads through fwa::b200::run_backbone
