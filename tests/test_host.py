"""Host-side logic on the CPU: the C-ABI library loads and exports every symbol the
header declares, the ctypes descriptor matches the C layout, host-only entry points
work, the Python mirror validates like the reference, and reference objects drop in."""

import ctypes
import re
import subprocess
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import paper_2310_00236_b200 as hw
from paper_2310_00236_b200 import _abi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "halfwave_b200.h"
REF_SRC = Path("/root/reference/pkg/src")


def header_functions():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|double|const char\*)\s+(hw_\w+)\(", txt, re.M)))


def test_library_exports_every_header_function():
    lib = _abi.load()
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(_abi.EXPORTED)
    assert b"sm_100a" in lib.hw_version()


def test_desc_layout_matches_c_header(tmp_path):
    fields = [f for f, _ in _abi.Desc._fields_]
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {",
           'printf("%zu\\n", sizeof(hw_desc));']
    src += [f'printf("%zu\\n", offsetof(hw_desc, {f}));' for f in fields]
    src += ["return 0; }"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(c)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_abi.Desc)
    for f, off in zip(fields, vals[1:]):
        assert getattr(_abi.Desc, f).offset == off, f


def test_host_only_entry_points():
    lib = _abi.load()
    assert lib.hw_num_fields(0, 2) == 6 and lib.hw_num_fields(0, 3) == 8
    assert lib.hw_num_fields(1, 2) == 10 and lib.hw_num_fields(1, 3) == 18
    g = hw.GridSpec(16, 12, 0.05, 0.01, 5, bc_y=hw.Boundary.FREE_SURFACE)
    s = hw.ElasticSolver(g, hw.build_layered_elastic(16, 12, [(1.0, 1.0, 2.0, 1.0)]))
    shape = (ctypes.c_int64 * 3)()
    for j, name in enumerate(s.FIELDS):
        assert lib.hw_field_shape(ctypes.byref(s.desc), j, shape) == 0
        assert (shape[0], shape[2]) == s.grid.shape(s._stagger_of(name))


def test_no_cpu_fallback_without_a_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    s = hw.AcousticSolver(hw.GridSpec(16, 16, 0.05, 0.01, 2), hw.build_homogeneous_acoustic(16, 16, 1.0, 1.0))
    with pytest.raises(RuntimeError, match="hw_create"):
        s.run()


def test_round_fraction_matches_exact_nearest():
    rng = np.random.default_rng(0)
    for p, fmt in ((hw.Precision.FP16, np.float16), (hw.Precision.FP32, np.float32)):
        for _ in range(3000):
            q = Fraction(int(rng.integers(-10**6, 10**6)), int(rng.integers(100, 10**7)))
            got = hw.round_fraction(p, q)
            # nearest representable, ties to even: compare with neighbours
            cand = float(fmt(float(q)))
            lo, hi = np.nextafter(fmt(cand), fmt(-np.inf)), np.nextafter(fmt(cand), fmt(np.inf))
            best = min((abs(Fraction(float(v)) - q), float(v)) for v in (fmt(cand), lo, hi) if np.isfinite(v))
            assert abs(Fraction(got) - q) == best[0]


def test_grid_and_solver_validation_messages():
    with pytest.raises(ValueError, match="at least 8"):
        hw.GridSpec(4, 16, 0.1, 0.01, 1)
    with pytest.raises(ValueError, match="periodic"):
        hw.GridSpec(16, 16, 0.1, 0.01, 1, bc_x=hw.Boundary.FREE_SURFACE)
    g = hw.GridSpec(16, 16, 0.032, float(np.float16(4e-4)), 10)
    m = hw.build_homogeneous_acoustic(16, 16, 1.0, 1.0)
    with pytest.raises(ValueError, match="periodic"):
        hw.AcousticSolver(hw.GridSpec(16, 16, 0.032, 0.0004, 10, bc_y=hw.Boundary.FREE_SURFACE), m)
    with pytest.raises(ValueError, match="acoustic medium"):
        hw.AcousticSolver(g, hw.build_layered_elastic(16, 16, [(1.0, 2.0, 3.0, 1.5)]))
    with pytest.raises(ValueError, match="pressure point"):
        hw.AcousticSolver(g, m, hw.SourceSpec(hw.SourceKind.VY_POINT, 2, 2, hw.RickerSpec(5.0)))
    with pytest.raises(ValueError, match="outside"):
        hw.AcousticSolver(g, m, receivers=((16, 0),))
    with pytest.raises(ValueError, match="energy_every"):
        hw.AcousticSolver(g, m, energy_every=0)
    with pytest.raises(ValueError, match="CFL"):
        hw.AcousticSolver(hw.GridSpec(16, 16, 0.032, 0.032, 10), m)
    with pytest.raises(ValueError, match="vertical-velocity"):
        hw.ElasticSolver(g, hw.build_layered_elastic(16, 16, [(1.0, 1.0, 2.0, 1.0)]),
                         hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 2, 2, hw.RickerSpec(5.0)))


def test_layered_acoustic_planes_sample_their_staggers():
    m = hw.build_layered_acoustic(8, 10, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    # rows at y = j/10 (cells, x faces) or (j + 1/2)/10 (y faces); interface at 0.5
    assert list(m.planes["rho_x"][:, 0]) == [1.0] * 5 + [1.5] * 5
    assert list(m.planes["rho_y"][:, 0]) == [1.0] * 5 + [1.5] * 5
    np.testing.assert_allclose(m.planes["beta"][:, 3], [1.0] * 5 + [1 / 2.25] * 5)
    assert m.c_max() == pytest.approx(1.5)


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference not mounted")
def test_reference_objects_drop_in_and_build_the_same_descriptor():
    sys.path.insert(0, str(REF_SRC))
    try:
        import halfwave as ref
    finally:
        sys.path.remove(str(REF_SRC))
    kw = dict(stencil_precision=ref.Precision.FP16, receivers=((3, 4), (10, 2)), energy_every=5)
    rg = ref.GridSpec(24, 20, 0.05, 0.01, 30, bc_y=ref.Boundary.FREE_SURFACE)
    rm = ref.build_layered_elastic(24, 20, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    rs = ref.SourceSpec(ref.SourceKind.VY_POINT, 12, 5, ref.RickerSpec(5.0, amplitude=20.0))
    a = hw.ElasticSolver(rg, rm, rs, **kw)
    mg = hw.GridSpec(24, 20, 0.05, 0.01, 30, bc_y=hw.Boundary.FREE_SURFACE)
    mm = hw.build_layered_elastic(24, 20, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    ms = hw.SourceSpec(hw.SourceKind.VY_POINT, 12, 5, hw.RickerSpec(5.0, amplitude=20.0))
    b = hw.ElasticSolver(mg, mm, ms, stencil_precision=hw.Precision.FP16, receivers=((3, 4), (10, 2)), energy_every=5)
    for f, _ in _abi.Desc._fields_:
        if f in ("plane", "receivers"):
            continue
        va, vb = getattr(a.desc, f), getattr(b.desc, f)
        if f == "taps":
            va, vb = list(va), list(vb)
        assert va == vb, f
    for pid in a._keep:
        np.testing.assert_array_equal(a._keep[pid], b._keep[pid])
    np.testing.assert_array_equal(a.source_samples(0, 30), b.source_samples(0, 30))
    # taps and source samples equal the reference's own objects
    assert tuple(a.stencil.coefficients) == ref.stencil.StencilSpec.make(ref.Precision.FP16, 0.05).coefficients
    for n in range(30):
        assert a.source_samples(n, 1)[0] == ref.sources.sample_source(rs, n * 0.01)
