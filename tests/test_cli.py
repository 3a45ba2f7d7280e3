"""Quokka CLI mirror (reference pkg/tests/test_cli.py:55-106)."""
import numpy as np
import pytest

from conftest import EXAMPLE_OPTIMIZED
from paper_2406_14084_b200.cli import scan_optimized, sim_main


def _ini(tmp_path, total, rank, buffer_q):
    path = tmp_path / "cfg.ini"
    path.write_text(f"[system]\ntotal_qbit={total} // Total qubit for simulation\n"
                    f"rank_qbit={rank}\nbuffer_qbit={buffer_q}\n")
    return str(path)


def test_unknown_config_key(tmp_path, capsys):
    circ = tmp_path / "h.txt"
    circ.write_text("1\nH 0 0\n")
    ini = tmp_path / "bad.ini"
    ini.write_text("[system]\ntotal_qbit=2\nrank_qbit=0\nbuffer_qbit=2\nextra=1\n")
    assert sim_main(["-i", str(ini), "-c", str(circ)]) == 1
    assert "extra" in capsys.readouterr().err


def test_missing_file(tmp_path, capsys):
    ini = _ini(tmp_path, 2, 0, 2)
    assert sim_main(["-i", ini, "-c", str(tmp_path / "nope.txt")]) == 1
    assert "cannot read" in capsys.readouterr().err


def test_layout_mismatch(tmp_path, capsys):
    opt = tmp_path / "opt.txt"
    opt.write_text(EXAMPLE_OPTIMIZED)
    ini = _ini(tmp_path, 10, 4, 6)
    assert sim_main(["-i", ini, "-c", str(opt)]) == 1
    err = capsys.readouterr().err
    assert "local" in err or "rank" in err


def test_scan_and_bad_structure(tmp_path, capsys):
    assert scan_optimized(EXAMPLE_OPTIMIZED) == (3, 8)
    bad = tmp_path / "bad.txt"
    bad.write_text("x\nH 0 0\n")
    assert sim_main(["-i", _ini(tmp_path, 2, 0, 2), "-c", str(bad)]) == 1
    assert "bad optimized circuit structure" in capsys.readouterr().err


@pytest.mark.gpu
def test_sim_runs_example(gpu, tmp_path, capsys):
    opt = tmp_path / "opt.txt"
    opt.write_text(EXAMPLE_OPTIMIZED)
    assert sim_main(["-i", _ini(tmp_path, 10, 2, 6), "-c", str(opt)]) == 0
    out = capsys.readouterr().out
    assert "norm 1.000000000000" in out
    for key in ("gate_seconds", "ims_seconds", "xrs_seconds", "aio_seconds"):
        assert key in out


@pytest.mark.gpu
def test_sim_amplitude_dump(gpu, tmp_path, capsys):
    circ = tmp_path / "h.txt"
    circ.write_text("1\nH 0 0\n")
    amps = tmp_path / "amps.txt"
    assert sim_main(["-i", _ini(tmp_path, 2, 0, 2), "-c", str(circ), "--amps", "4",
                     "--amps-file", str(amps)]) == 0
    vals = [complex(float(a), float(b)) for a, b in
            (line.split() for line in amps.read_text().splitlines())]
    assert np.allclose(vals, [2 ** -0.5, 2 ** -0.5, 0, 0])
    assert sim_main(["-i", _ini(tmp_path, 2, 0, 2), "-c", str(circ), "--amps", "2"]) == 0
    out = capsys.readouterr().out
    assert "amp 0 0.7071067811865475 0.0" in out or "amp 0 0.7071067811865476 0.0" in out
