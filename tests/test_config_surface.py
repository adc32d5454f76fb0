"""CPU: the reference's configuration surface on the host mirror
(paper_2507_07120_b200/model.py): ParallelismConfig / HardwareSpec /
validate_config / load_hardware with the reference's JSON schema and rules.

validate_config is pinned to the REFERENCE ITSELF: tests/golden/validate_config.json
holds what the reference's own validate_config (types.cpp:86-141, compiled
from /root/reference by oracle/Makefile, generator oracle/gen_config_golden.cpp)
returns over 2880 layouts x models (GQA, MLA, MoE, MoE with non-dividing
widths) -- verdict and first-broken-rule text must match exactly."""
import json
import os

import pytest

from paper_2507_07120_b200 import model as M

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "validate_config.json")


def _models():
    gqa = M.ModelSpec("gqa", 2, 16384, 128, 8, 128, 65536, 3, "gqa", 0)
    mla = M.ModelSpec("mla", 2, 16384, 128, 1, 128, 65536, 3, "mla", 288)
    moe = M.ModelSpec("moe", 2, 16384, 128, 8, 128, 65536, 3, "gqa", 0, M.MoESpec(256, 8, 2048, 2048))
    odd = M.ModelSpec("moe_odd", 2, 16384, 128, 8, 128, 65536, 3, "gqa", 0, M.MoESpec(6, 2, 24, 0))
    return {m.name: m for m in (gqa, mla, moe, odd)}


def test_validate_config_matches_reference_golden():
    g = json.load(open(GOLDEN))
    cols = g["columns"]
    models = _models()
    for row in g["rows"]:
        r = dict(zip(cols, row))
        hw = M.HardwareSpec(max_gpus=r["max_gpus"])
        cfg = M.ParallelismConfig(r["strategy"], r["tpa"], r["kvp"], r["tpf"], r["ep"], r["pp"])
        v = M.validate_config(cfg, models[r["model"]], hw)
        assert (bool(v), v.rule, cfg.total_gpus()) == (bool(r["ok"]), r["rule"], r["total_gpus"]), r


def test_hardware_presets_round_trip_and_reference_files():
    hw = M.load_hardware("gb200-like")
    assert M.HardwareSpec.from_json(hw.to_json()) == hw
    ref = "/root/reference/proj/presets/gb200-like.json"
    if os.path.exists(ref):  # the reference's own preset file parses to the same values
        assert M.load_hardware(ref) == hw
    b200 = M.load_hardware("b200-measured")
    assert b200.bytes_per_param == 2.0 and b200.max_gpus == 8


@pytest.mark.parametrize("bad,msg", [
    ({"name": "x"}, "missing field"),
    ({**M.HARDWARE_PRESETS["gb200-like"].to_json(), "extra": 1}, "unknown key 'extra'"),
    ({**M.HARDWARE_PRESETS["gb200-like"].to_json(), "max_gpus": 1.5}, "must be an integer"),
])
def test_hardware_json_errors(bad, msg):
    with pytest.raises(M.ConfigError, match=msg):
        M.HardwareSpec.from_json(bad)


def test_parallelism_json_schema():
    cfg = M.ParallelismConfig("helix", 1, 8, 8, 1, 1)
    assert M.ParallelismConfig.from_json(cfg.to_json()) == cfg
    assert str(cfg) == "helix(tpa=1,kvp=8,tpf=8,ep=1,pp=1)"
    with pytest.raises(M.ConfigError, match="unknown value 'bogus'"):
        M.ParallelismConfig.from_json({**cfg.to_json(), "strategy": "bogus"})
    with pytest.raises(M.ConfigError, match="unknown key 'x'"):
        M.ParallelismConfig.from_json({**cfg.to_json(), "x": 1})


def test_from_config_rejects_invalid_layouts_before_touching_the_gpu():
    spec = M.PRESETS["llama405b-like"]
    with pytest.raises(ValueError, match="kvp\\*tpa must equal tpf\\*ep"):
        M.HelixDecoder.from_config(spec, M.ParallelismConfig("helix", 1, 8, 4, 1, 1))
    with pytest.raises(ValueError, match="helix strategy"):
        M.HelixDecoder.from_config(spec, M.ParallelismConfig("tp", 8, 1, 8, 1, 1))


def test_cpp_config_surface_matches_reference():
    """include/helixsim/config_b200.hpp (the C++ L0/L1 surface: specs, JSON
    schema, presets, validate_config, lowering onto the C ABI) -- the C++
    test tests/cpp/test_config_b200.cpp against the same reference golden."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call(["make", "-s", "-C", os.path.join(root, "tests", "cpp"), "test_config_b200"])
    env = dict(os.environ, HX_GOLDEN_DIR=os.path.join(root, "tests", "golden"))
    if os.path.isdir("/root/reference/proj/presets"):
        env["HX_REF_PRESETS"] = "/root/reference/proj/presets"
    out = subprocess.run([os.path.join(root, "tests", "cpp", "test_config_b200")], capture_output=True, text=True,
                         env=env, timeout=120)
    assert out.returncode == 0, out.stdout[-3000:]
    assert "failed: 0" in out.stdout.splitlines()[-1]
