"""The C oracle against the unmodified reference at BASELINE config 1's full size and length
(the reference-native 4th-order periodic twins, tests/golden/twin/): final field bits (SHA-256),
traces bit for bit, the 2001-sample energy history within 1e-12 -- and the reference's own
finding that compensation helps at CFL 0.05 / 0.0125 but not at the configured CFL 0.5."""

import numpy as np
import pytest

import oracle
from twin_cases import Twin, names, relative_change


@pytest.mark.parametrize("name", names())
def test_oracle_matches_reference_twin(name):
    tw = Twin(name)
    solver = tw.solver()
    st = tw.initial_state(solver)
    out = oracle.run_solver(solver, tw.variant, st)
    assert out["fail"] is None
    tw.check(out["fields"], out["traces"], out["e_times"], out["e_vals"])


def test_reference_twin_energy_behaviour():
    """BASELINE.md 'Energy behaviour at config 1's CFL' from the fixtures themselves."""
    e = {n: Twin(n).z["e_vals"] for n in names()}
    assert abs(relative_change(e["twin_cfl0p5_fp64_naive"])) < 1e-12
    # CFL 0.5: binary16 stencil rounding dominates; op3 is no better than naive
    assert abs(relative_change(e["twin_cfl0p5_fp16_op3"])) > abs(relative_change(e["twin_cfl0p5_fp16_naive"]))
    # CFL 0.05 and 0.0125: the naive update swamps (energy decays), compensation recovers >= 100x
    for c in ("0p05", "0p0125"):
        naive, op3 = relative_change(e[f"twin_cfl{c}_fp16_naive"]), relative_change(e[f"twin_cfl{c}_fp16_op3"])
        assert naive < -5e-3
        assert abs(op3) < abs(naive) / 100
    assert len(np.unique([len(v) for v in e.values()])) == 1
