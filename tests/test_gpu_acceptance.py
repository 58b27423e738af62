"""The reference's energy-behaviour acceptance gate (pkg/tests/test_acceptance.py:165-255,
criteria 4-8) on the B200 path.

The reference's desk runs (paper-acoustic / paper-elastic presets at desk scale, in every
precision mode the criteria interrogate) were run UNMODIFIED and kept as fixtures
(tests/golden/make_acceptance_golden.py -> tests/golden/acceptance/).  Here
  * (CPU) the fixtures themselves pass criteria 4-8 through this package's mirror of
    diagnostics.energy_drift / compare_traces (diagnostics.py:56-91), the reference thresholds
    unchanged (wall-time budgets dropped);
  * (GPU) the same desk runs through SimConfig.run() on the device reproduce every fixture
    (traces bit for bit, energy histories within 1e-12) and pass the same criteria.
So the naive-vs-compensated energy behaviour the paper reports is the reference's, on the GPU.
"""
from pathlib import Path

import numpy as np
import pytest

from paper_2310_00236_b200 import config
from paper_2310_00236_b200.diagnostics import EnergySeries, compare_traces, energy_drift

GOLD = Path(__file__).resolve().parent / "golden" / "acceptance"
ACOUSTIC = {"fp64": ("fp64", "fp64", "baseline"), "fp16-base": ("fp16", "fp16", "baseline"),
            "fp16-op3": ("fp16", "fp16", "op3"), "mixed-naive": ("fp64", "fp16", "baseline"),
            "mixed-op3": ("fp64", "fp16", "op3")}
ELASTIC = {"fp64": ("fp64", "fp64", "baseline"), "fp16-base": ("fp16", "fp16", "baseline"),
           "fp16-op6": ("fp16", "fp16", "op6"), "fp16-op3": ("fp16", "fp16", "op3")}
RUNS = [("paper-acoustic", n) for n in ACOUSTIC] + [("paper-elastic", n) for n in ELASTIC]


class Run:
    """Traces and energy history of one desk run (fixture or device)."""

    def __init__(self, traces, e_times, e_vals, t_off):
        self.traces = [np.asarray(t, dtype=np.float64) for t in traces]
        self.energy = EnergySeries(np.asarray(e_times, dtype=np.float64), np.asarray(e_vals, dtype=np.float64))
        self.t_off = float(t_off)


def _fixture(preset, name):
    z = np.load(GOLD / f"{preset}_{name}.npz")
    return Run(z["traces"], z["e_times"], z["e_vals"], z["t_source_off"])


def _cfg(preset, name):
    s, u, m = (ACOUSTIC if preset == "paper-acoustic" else ELASTIC)[name]
    return config.parse_config(preset=preset, desk=True,
                               sets=[f"precision.stencil={s}", f"precision.update={u}", f"precision.mode={m}"])


_DEVICE = {}


def _device(preset, name):
    if (preset, name) not in _DEVICE:
        cfg = _cfg(preset, name)
        out = cfg.run()
        _DEVICE[(preset, name)] = Run([t.samples for t in out.traces], out.energy.times, out.energy.values,
                                      2.0 * cfg.source.wavelet.delay)
    return _DEVICE[(preset, name)]


def _criteria(get):
    """Criteria 4-8 (test_acceptance.py:165-255) on runs from get(preset, name); returns the
    measured values, asserting each criterion."""
    a = lambda n: get("paper-acoustic", n)  # noqa: E731
    e = lambda n: get("paper-elastic", n)  # noqa: E731
    m = {}
    ref = a("fp64")
    m["c4_fp64_dev"] = energy_drift(ref.energy, ref.t_off)["rel_deviation"]
    assert m["c4_fp64_dev"] <= 1e-10, m
    d = energy_drift(a("fp16-base").energy, ref.t_off)
    m["c5_naive_dev"], m["c5_naive_slope"] = d["rel_deviation"], d["trend_slope"]
    assert m["c5_naive_dev"] >= 1e-2 and m["c5_naive_slope"] < 0.0, m
    e_ref = float(ref.energy.values[-1])
    m["c6_op3_final_rel"] = abs(float(a("fp16-op3").energy.values[-1]) - e_ref) / abs(e_ref)
    m["c6_trace_op3"] = compare_traces(a("fp16-op3").traces[0], ref.traces[0])["l2_rel"]
    m["c6_trace_naive"] = compare_traces(a("fp16-base").traces[0], ref.traces[0])["l2_rel"]
    assert m["c6_op3_final_rel"] <= 1e-2 and m["c6_trace_op3"] <= m["c6_trace_naive"] / 5.0, m
    m["c7_mixed_naive_dev"] = energy_drift(a("mixed-naive").energy, ref.t_off)["rel_deviation"]
    m["c7_mixed_op3_final_rel"] = abs(float(a("mixed-op3").energy.values[-1]) - e_ref) / abs(e_ref)
    assert m["c7_mixed_naive_dev"] > 1e-10 and m["c7_mixed_op3_final_rel"] <= 1e-2, m
    eref = e("fp64")
    m["c8_fp64_dev"] = energy_drift(eref.energy, eref.t_off)["rel_deviation"]
    m["c8_naive_dev"] = energy_drift(e("fp16-base").energy, eref.t_off)["rel_deviation"]
    ee = float(eref.energy.values[-1])
    m["c8_op6_final_rel"] = abs(float(e("fp16-op6").energy.values[-1]) - ee) / abs(ee)
    h3, h6 = e("fp16-op3").energy.values, e("fp16-op6").energy.values
    m["c8_variant_gap"] = float(np.max(np.abs(h3 - h6)) / np.max(np.abs(h6)))
    assert (m["c8_fp64_dev"] <= 1e-8 and m["c8_naive_dev"] >= 1e-2 and m["c8_op6_final_rel"] <= 1e-2
            and m["c8_variant_gap"] <= 1e-3), m
    return m


def test_reference_fixtures_pass_acceptance_criteria():
    """Pins the fixtures and the diagnostics mirror: the reference's own desk outputs pass
    criteria 4-8 when evaluated with this package's energy_drift / compare_traces."""
    m = _criteria(_fixture)
    assert m["c5_naive_dev"] > 100 * m["c6_op3_final_rel"]


@pytest.mark.gpu
@pytest.mark.parametrize("preset,name", RUNS)
def test_gpu_desk_run_reproduces_reference(preset, name):
    got, want = _device(preset, name), _fixture(preset, name)
    assert len(got.traces) == len(want.traces)
    for a, b in zip(got.traces, want.traces):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(got.energy.times, want.energy.times)
    np.testing.assert_allclose(got.energy.values, want.energy.values, rtol=1e-12)


@pytest.mark.gpu
def test_gpu_desk_runs_pass_acceptance_criteria():
    m = _criteria(_device)
    ref = _criteria(_fixture)
    for k in m:  # the same measured values as the reference's runs (to the energy tolerance; the fp64
        # flatness figures are ~1e-14 and move with the 1e-12 energy agreement)
        assert m[k] == pytest.approx(ref[k], rel=1e-6, abs=(1e-11 if "fp64_dev" in k else 1e-15)), k
