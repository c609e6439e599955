"""CLI device path: flag/config layering and exit codes (CPU: error paths only)."""

import subprocess
import sys

import pytest

from paper_2009_12638_b200.cli import boundary_from, main, read_config_file
from paper_2009_12638_b200.errors import ConfigurationError


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


@pytest.mark.gpu
def test_cli_run_exit_codes_and_trace(tmp_path):
    out = tmp_path / "t.csv"
    code = main(["run", "--nx", "8", "--ny", "8", "--nz", "8", "--gz", "2", "--inner", "cg", "--inner-its", "10",
                 "--tol", "1e-6", "--out", str(out)])
    assert code == 0 and out.read_text().startswith("outer_iteration,time,")
    code = main(["run", "--nx", "8", "--ny", "8", "--nz", "8", "--gz", "2", "--inner", "cg", "--inner-its", "2",
                 "--tol", "1e-12", "--max-outer", "3", "--out", str(out)])
    assert code == 2
