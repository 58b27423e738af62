"""BASELINE config 1's reference-native twins on the B200 at full size and length (256^2,
4th-order periodic, 2000 steps, energy every step, CFL 0.5 / 0.05 / 0.0125; fp16 naive, fp16
op3, fp64): the persistent small-grid kernel (fp16) and the generic kernels (fp64) reproduce
the UNMODIFIED reference's final field bits, traces and energy history (1e-12)."""

import pytest

import paper_2310_00236_b200 as hw
from twin_cases import FIELDS, Twin, names

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", names())
def test_gpu_matches_reference_twin(name):
    tw = Twin(name)
    solver = tw.solver()
    st = tw.initial_state(solver)
    out = solver.run(tw.variant, st)
    assert solver.kernel_path() == ("small2d" if tw.d["precision"] == "fp16" else "generic")
    assert st.step == tw.d["nt"]
    tw.check([getattr(st, n).values for n in FIELDS], [t.samples for t in out.traces], out.energy.times,
             out.energy.values)
