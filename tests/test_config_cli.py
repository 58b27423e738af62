"""Config / CLI / WMED layer (SURVEY §8 f): same schema, presets, overrides, errors and
output formats as the reference's config.py / cli.py, driving the B200 solvers."""

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2310_00236_b200 as hw
from paper_2310_00236_b200 import cli, config
from paper_2310_00236_b200.grids import load_medium, save_medium

ROOT = Path(__file__).resolve().parents[1]
GOLD = Path(__file__).resolve().parent / "golden" / "cli"
REF_SRC = Path("/root/reference/pkg/src")


def test_presets_and_desk_scaling():
    c = config.parse_config(preset="paper-acoustic", desk=True)
    assert (c.grid.nx, c.grid.ny, c.grid.nt, c.grid.dx) == (150, 150, 6000, 0.032)
    assert c.grid.dt == config.DT16 and c.receivers == ((66, 66),)
    assert c.label == "paper-acoustic-desk" and c.variant is hw.Variant.OP3
    assert c.stencil_precision is hw.Precision.FP16 and c.equation == "acoustic"
    e = config.parse_config(preset="paper-elastic", desk=True, sets=["precision.mode=op3"])
    assert e.grid.free_surface_y and e.variant is hw.Variant.OP3 and e.source.kind is hw.SourceKind.VY_POINT


@pytest.mark.parametrize("sets,match", [
    (["grid.bogus=1"], "unknown key"), (["nosection.x=1"], "unknown key"), (["grid.nx"], "section.key=value"),
    (["precision.mode=op9"], "precision.mode"), (["grid.nx=abc"], "cannot parse"),
    (["grid.dt=1.0"], "CFL"), (["receivers.points=500 5"], "outside"),
])
def test_config_errors(sets, match):
    with pytest.raises(ValueError, match=match):
        config.parse_config(preset="paper-acoustic", desk=True, sets=sets)


def test_ini_file_with_extensions(tmp_path):
    ini = tmp_path / "x.ini"
    ini.write_text("[grid]\nnx = 32\nny = 16\nnz = 24\ndx = 0.05\ndt = 0.01\nnt = 5\norder = 2\n"
                   "[medium]\nkind = acoustic\nlayers = 0.5 1.0 1.0; 1.0 1.5 2.25\n"
                   "[source]\nkind = pressure-point\nix = 3\niy = 4\niz = 5\nf_center = 5\n"
                   "[receivers]\npoints = 1 2 3; 4 5 6\n[precision]\nstencil = fp16\nmode = op3\n"
                   "[run]\nslabs = 2  # two slabs on one device\n")
    c = config.parse_config(ini)
    assert c.grid.nz == 24 and c.grid.order == 2 and c.slabs == 2
    assert c.medium.ndim == 3 and c.receivers == ((1, 2, 3), (4, 5, 6)) and c.source.iz == 5
    with pytest.raises(ValueError, match="exactly one"):
        config.parse_config(ini, preset="paper-acoustic")


def test_wmed_round_trip_and_errors(tmp_path):
    m = hw.build_layered_elastic(12, 10, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    p = tmp_path / "m.wmed"
    save_medium(p, m)
    back = load_medium(p)
    for k in m.planes:
        np.testing.assert_array_equal(back.planes[k], m.planes[k])
    raw = p.read_bytes()
    (tmp_path / "bad.wmed").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="magic"):
        load_medium(tmp_path / "bad.wmed")
    (tmp_path / "short.wmed").write_bytes(raw[:-8])
    with pytest.raises(ValueError, match="size mismatch"):
        load_medium(tmp_path / "short.wmed")


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference not mounted")
def test_wmed_files_interoperate_with_the_reference(tmp_path):
    sys.path.insert(0, str(REF_SRC))
    try:
        import halfwave
    finally:
        sys.path.remove(str(REF_SRC))
    rm = halfwave.build_layered_elastic(12, 10, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    halfwave.save_medium(tmp_path / "r.wmed", rm)
    mine = load_medium(tmp_path / "r.wmed")
    save_medium(tmp_path / "m.wmed", mine)
    assert (tmp_path / "m.wmed").read_bytes() == (tmp_path / "r.wmed").read_bytes()
    # formats table and audit agree with the reference CLI
    from halfwave.cli import formats_table, range_audit
    assert cli.formats_table() == formats_table()
    rc = halfwave.config.parse_config(None, preset="paper-elastic", desk=True)
    mc = config.parse_config(preset="paper-elastic", desk=True)
    ref_lines = range_audit(rc).render().splitlines()
    got = [l for l in cli.range_audit(mc).render().splitlines() if "SURVEY" not in l]
    if ref_lines == ["range audit: all values inside the normal range"]:
        assert got == [] or got == ref_lines
    else:
        assert got == ref_lines


def test_audit_flags_overflowing_divisors_and_tap_headroom():
    c = config.parse_config(preset="paper-acoustic", desk=True, sets=["medium.rho=1e-9"])
    rep = cli.range_audit(c)
    assert not rep.ok and "rounds to zero" in rep.render()
    ok = config.parse_config(preset="paper-acoustic", desk=True)
    assert cli.range_audit(ok).ok and "tap products overflow" in cli.range_audit(ok).render()


def test_cli_usage_errors_and_formats():
    assert cli.main(["formats"]) == 0
    assert cli.main(["audit", "--preset", "paper-acoustic", "--desk"]) == 0
    assert cli.main(["run", "--preset", "paper-acoustic", "--desk", "--set", "grid.nx=abc"]) == 2
    assert cli.main(["audit", "--preset", "paper-acoustic", "--desk", "--set", "medium.rho=1e-9"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["paper-acoustic", "paper-elastic"])
def test_cli_desk_run_matches_reference_outputs(tmp_path, preset):
    """`run --preset X --desk` on the B200: traces.csv byte-identical to the reference
    CLI's; energy.csv times identical and energies within 1e-12."""
    r = subprocess.run([sys.executable, "-m", "paper_2310_00236_b200.cli", "run", "--preset", preset, "--desk",
                        "--out", str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = tmp_path / f"{preset}-desk"
    assert (out / "traces.csv").read_bytes() == (GOLD / preset / "traces.csv").read_bytes()
    got = np.loadtxt(out / "energy.csv", delimiter=",", skiprows=1)
    want = np.loadtxt(GOLD / preset / "energy.csv", delimiter=",", skiprows=1)
    np.testing.assert_array_equal(got[:, 0], want[:, 0])
    np.testing.assert_allclose(got[:, 1], want[:, 1], rtol=1e-12)


@pytest.mark.gpu
def test_cli_mid_run_range_failure_matches_reference(tmp_path):
    """A run that passes the static audit and goes non-finite mid-wavelet (reference behaviour:
    test_cli.py:311-327): same exit code, same failing step and field in summary.json as the
    reference CLI on the same INI file (tests/golden/cli/range-failure/, make_cli_golden.py)."""
    import json

    gold = GOLD / "range-failure"
    r = subprocess.run([sys.executable, "-m", "paper_2310_00236_b200.cli", "run", "--config", str(gold / "case.ini"),
                        "--out", str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == int((gold / "exit_code.txt").read_text()) == 1
    got = json.loads((tmp_path / "overdrive" / "summary.json").read_text())
    want = json.loads((gold / "summary.json").read_text())
    assert got["range_failure"] == want["range_failure"] == {"field": "Vy", "step": 83}
    assert "non-finite" in r.stderr


def test_ini_rigid_walls(tmp_path):
    """grid.bc_x / grid.bc_y = rigid (p = 0 walls, extension) parse into a rigid GridSpec."""
    ini = tmp_path / "box.ini"
    ini.write_text("[grid]\nnx = 32\nny = 24\ndx = 0.03125\ndt = 0.005\nnt = 4\norder = 2\nbc_x = rigid\nbc_y = rigid\n"
                   "[medium]\nkind = acoustic\nrho = 1.0\nc = 1.0\n[precision]\nstencil = fp16\nmode = op3\n")
    c = config.parse_config(ini)
    assert c.grid.rigid_x and c.grid.rigid_y and c.grid.shape(hw.Stagger.CELL) == (25, 33)
    with pytest.raises(ValueError, match="periodic"):
        config.parse_config(ini, sets=["grid.bc_x=free-surface"])
