"""CLI device path (cli.py of the reference, 263-586): flag/config layering,
exit codes, the ``sweep`` and ``compare`` subcommands, and trace parity with
golden outputs of the reference's own CLI (tests/golden/make_cli_golden.py).

CPU: parsing, error paths and ``compare`` (pure CSV work) against the
reference's table and CSV byte for byte.  GPU: ``run`` / ``sweep`` traces
field by field against the reference's."""

import json
import os
import shutil

import pytest

from paper_2009_12638_b200.cli import axis_values, boundary_from, main, read_config_file
from paper_2009_12638_b200.errors import ConfigurationError
from paper_2009_12638_b200.multisplit import ResidualTrace

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def _meta():
    with open(os.path.join(GOLD, "cli_golden.json")) as fh:
        return json.load(fh)


def test_boundary_parsing():
    b = boundary_from("faces:x_lo=1,y_hi=0.5")
    assert b.face_constants()["x_lo"] == 1.0 and b.face_constants()["y_hi"] == 0.5
    assert boundary_from("const:2").face_constants()["z_hi"] == 2.0
    with pytest.raises(ConfigurationError):
        boundary_from("faces:w_lo=1")
    with pytest.raises(ConfigurationError):
        boundary_from("nonsense")


def test_config_file_and_errors(tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text("# comment\nnx=4\nmode=sync\n")
    assert read_config_file(str(p)) == {"nx": "4", "mode": "sync"}
    bad = tmp_path / "bad.cfg"
    bad.write_text("nx 4\n")
    with pytest.raises(ConfigurationError):
        read_config_file(str(bad))
    # unknown key / invalid mode -> exit code 1 (cli.py:584-586), before any device work
    unk = tmp_path / "unk.cfg"
    unk.write_text("colour=blue\n")
    assert main(["run", "--config", str(unk)]) == 1
    assert main(["run", "--mode", "warp"]) == 1
    assert main(["run", "--nx", "abc"]) == 1
    assert main(["run", "--residual-mode", "fuzzy"]) == 1
    assert main(["run", "--exec", "fibers"]) == 1


def test_sweep_axis_parsing():
    assert axis_values("block_grid", "1,1,2;2,2,2") == [(1, 1, 2), (2, 2, 2)]
    assert axis_values("inner_max_its", "5,10,") == [5, 10]
    assert axis_values("mode", "sync,async") == ["sync", "async"]
    for axis, raw in (("block_grid", "1,2"), ("mode", "warp"), ("overlap", "x"), ("colour", "1")):
        with pytest.raises(ConfigurationError):
            axis_values(axis, raw)
    assert main(["sweep", "--axis", "colour", "--values", "1"]) == 1
    assert main(["sweep", "--axis", "block_grid", "--values", "1,2"]) == 1


def test_compare_matches_reference_cli(tmp_path, capsys):
    """``compare`` over the reference's own traces: the same table and the
    same CSV bytes as the reference's ``blocksolve compare``."""
    m = _meta()["compare"]
    for name in m["traces"]:
        shutil.copy(os.path.join(GOLD, name), tmp_path / name)
    cwd = os.getcwd()
    os.chdir(tmp_path)
    try:
        code = main(["compare"] + m["traces"] + ["--reference", m["reference"], "--out", "cmp.csv"])
        out = capsys.readouterr().out
    finally:
        os.chdir(cwd)
    assert code == m["code"] == 0
    assert out == m["stdout"]
    with open(os.path.join(GOLD, m["csv"])) as fh:
        assert (tmp_path / "cmp.csv").read_text() == fh.read()
    assert main(["compare", str(tmp_path / m["traces"][0]), "--reference", "missing.csv"]) == 1
    empty = tmp_path / "empty.csv"
    empty.write_text(open(os.path.join(GOLD, m["traces"][0])).readline())
    assert main(["compare", str(empty)]) == 1


def _assert_trace_matches(path, golden_path):
    got = ResidualTrace.read_csv(str(path)).rows
    ref = ResidualTrace.read_csv(golden_path).rows
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        assert (g.outer_iteration, g.time, g.inner_iterations, g.max_halo_staleness) == \
               (r.outer_iteration, r.time, r.inner_iterations, r.max_halo_staleness)
        # reassociated dots move a per-sweep residual by up to ~1e-12 absolute
        # (tests/test_oracle_envelope.py, the reference against itself)
        assert g.estimated_residual == pytest.approx(r.estimated_residual, rel=1e-9, abs=5e-12)
        assert (g.true_residual is None) == (r.true_residual is None)
        if r.true_residual is not None:
            assert g.true_residual == pytest.approx(r.true_residual, rel=1e-9, abs=5e-12)


@pytest.mark.gpu
def test_cli_run_trace_matches_reference(tmp_path, capsys):
    m = _meta()
    for key in ("run", "run_capped"):
        out = tmp_path / f"{key}.csv"
        code = main(["run"] + m[key]["argv"] + ["--out", str(out)])
        text = capsys.readouterr().out
        assert code == m[key]["code"]
        _assert_trace_matches(out, os.path.join(GOLD, m[key]["trace"]))
        # summary lines: counts exact, the residual printed to 6 digits
        got = dict((line[:24].strip(), line[24:]) for line in text.splitlines())
        ref = dict((line[:24].strip(), line[24:]) for line in m[key]["stdout"].splitlines())
        for field in ("outer iterations", "total inner iterations", "iteration rate", "converged"):
            assert got[field] == ref[field], field
        assert float(got["final true residual"]) == pytest.approx(float(ref["final true residual"]), rel=1e-5)


@pytest.mark.gpu
def test_cli_sweep_matches_reference(tmp_path, capsys):
    m = _meta()["sweep"]
    out = tmp_path / "sweep.csv"
    code = main(["sweep"] + m["argv"] + ["--out", str(out), "--summary-out", str(tmp_path / "summary.csv")])
    capsys.readouterr()
    assert code == m["code"]
    for name in m["traces"]:
        _assert_trace_matches(tmp_path / name, os.path.join(GOLD, name))
    got = (tmp_path / "summary.csv").read_text().splitlines()
    with open(os.path.join(GOLD, m["summary"])) as fh:
        ref = fh.read().splitlines()
    assert got[0] == ref[0] and len(got) == len(ref)
    for g, r in zip(got[1:], ref[1:]):
        g, r = g.split(","), r.split(",")
        assert g[:3] == r[:3] and g[4] == r[4]
        assert float(g[3]) == pytest.approx(float(r[3]), rel=1e-9, abs=5e-12)
