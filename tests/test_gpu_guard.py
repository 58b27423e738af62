"""The guarded device allocations (option "guard", HW_TEST_GUARD for the whole suite): an access one
byte outside a buffer faults instead of landing in a neighbouring allocation.  Each probe runs in a
process of its own (a fault loses the CUDA context)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
PROBE = ("import sys; sys.path.insert(0, {root!r}); import paper_2310_00236_b200 as hw; "
         "from paper_2310_00236_b200 import _abi; hw.set_option('guard', {guard}); "
         "rc = _abi.load().hw_selftest_guard(0, {off}); print('rc', rc); sys.exit(0 if rc == 0 else 3)")


def _probe(guard, off):
    r = subprocess.run([sys.executable, "-c", PROBE.format(root=str(ROOT), guard=guard, off=off)],
                       capture_output=True, text=True, timeout=300)
    return r.returncode


@pytest.mark.parametrize("guard,off", [(0, 0), (1, 0), (1, 4095), (2, 0), (2, 4095)])
def test_guarded_buffers_are_fully_accessible(guard, off):
    assert _probe(guard, off) == 0


@pytest.mark.skipif(os.environ.get("HW_GUARD_PROBE") != "1",
                    reason="deliberately raises a GPU MMU fault (Xid 31) in a child process: run with HW_GUARD_PROBE=1 "
                           "(green in this round's checkpoints, profiles/r2_gpu_tests.txt: 510 passed with both probes)")
@pytest.mark.parametrize("guard,off", [(1, -1), (2, 4096)])
def test_guard_catches_out_of_bounds(guard, off):
    """One byte before a start-aligned buffer / one byte past an end-aligned one faults."""
    assert _probe(guard, off) != 0


def test_solver_runs_under_guard(hwopt):
    """A fused-kernel run with every buffer guarded, both alignments (the whole suite: HW_TEST_GUARD)."""
    import numpy as np

    import paper_2310_00236_b200 as hw

    for g in (1, 2):
        hwopt(guard=g, small=0)
        n = 256
        s = hw.AcousticSolver(hw.GridSpec(n, 64, 1.0 / n, float(np.float16(0.3 / n)), 12),
                              hw.build_layered_acoustic(n, 64, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)]),
                              stencil_precision=hw.Precision.FP16, energy_every=3)
        st = s.new_state()
        st.p.values = np.random.default_rng(0).uniform(-1, 1, st.p.values.shape).astype(np.float16)
        out = s.run(hw.Variant.OP3, st)
        assert s.kernel_path() == "fused2d" and np.isfinite(out.energy.values).all()
        s.close()
