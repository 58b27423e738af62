"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The oracle (oracle/halfwave_oracle.c) is driven through this package's host
descriptor, so these tests also pin the host-side plumbing (taps, lane
constants, medium materialisation, source sampling, receivers) that the GPU
path shares.  Bit-exact fields and traces; energy within 1e-12 relative (the
reference's np.sum order is not part of its contract).
"""

import numpy as np
import pytest

import oracle
from golden_cases import Case, assert_same_bits, names

ENERGY_RTOL = 1e-12


@pytest.mark.parametrize("name", [n for n in names() if not Case(n).d["steps_api"]])
def test_oracle_run_matches_reference(name):
    case = Case(name)
    solver = case.solver()
    st = case.initial_state(solver)
    out = oracle.run_solver(solver, case.variant, st)
    want_fail = case.d.get("fail")
    if want_fail:
        assert out["fail"] is not None, "reference raised RangeFailureError, oracle did not"
        step, field = out["fail"]
        assert step == want_fail[0]
        assert solver._fail_name(field) == want_fail[1]
    else:
        assert out["fail"] is None
        np.testing.assert_array_equal(out["traces"], case.z["traces"])
        np.testing.assert_array_equal(out["e_times"], case.z["e_times"])
        np.testing.assert_allclose(out["e_vals"], case.z["e_vals"], rtol=ENERGY_RTOL, atol=0)
    for j, n in enumerate(solver.FIELDS):
        assert_same_bits(out["fields"][j], case.z[f"final_{n}"], f"{name}:{n}")


@pytest.mark.parametrize("name", [n for n in names() if Case(n).d["steps_api"]])
def test_oracle_single_steps_match_reference(name):
    case = Case(name)
    solver = case.solver()
    arrays = [case.z[f"init_{n}"] for n in solver.FIELDS]
    from paper_2310_00236_b200.efsum import variant_code

    for k in range(case.d["steps_api"]):
        src = solver.source_samples(k, 1)
        out = oracle.run_desc(solver.desc, arrays, variant_code(case.variant), k, 1, src, energy=False)
        for j, n in enumerate(solver.FIELDS):
            assert_same_bits(out["fields"][j], case.z[f"step{k}_{n}"], f"{name}: step {k} {n}")
        arrays = out["fields"]


def test_oracle_round_lane_matches_numpy_casts():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(200_000) * np.exp2(rng.uniform(-30, 17, 200_000)),
        [0.0, -0.0, np.inf, -np.inf, 65504.0, 65519.99, 65520.0, 2.0 ** -25, 2.0 ** -24 * 1.5, 1e-30],
    ])
    # every binary16 midpoint (exact ties) and its neighbours
    h = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = (h[:-1] + h[1:]) / 2
    x = np.concatenate([x, mids, -mids, np.nextafter(mids, 0), np.nextafter(mids, 1e9)])
    with np.errstate(over="ignore"):
        want16 = x.astype(np.float16).astype(np.float64)
        want32 = x.astype(np.float32).astype(np.float64)
    np.testing.assert_array_equal(oracle.round_lane(16, x), want16)
    np.testing.assert_array_equal(oracle.round_lane(32, x), want32)
    np.testing.assert_array_equal(oracle.round_lane(64, x), x)
