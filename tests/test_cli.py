"""CLI (`qcsim run --mode full` mirror) and QSVDUMP I/O."""

import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2008_07140_b200 import cli


def test_format_pmeasure_matches_reference(golden, golden_arrays):
    for name, text in golden["format_pmeasure"].items():
        assert cli.format_pmeasure(golden_arrays[f"run/{name}/table0"]) == text, name


def test_rqc_command_byte_identical(golden, tmp_path, capsys):
    rec = golden["rqc"][1]
    assert cli.main(["rqc", "--rows", str(rec["rows"]), "--cols", str(rec["cols"]), "--depth",
                     str(rec["depth"]), "--seed", str(rec["seed"])]) == 0
    assert capsys.readouterr().out == rec["text"]


def test_error_exit_codes_and_log_lines(golden, tmp_path):
    for name, rec in golden["errors"].items():
        if rec["stage"] != "parse" and rec.get("error") != "TooManyQubits":
            continue
        script = tmp_path / f"{name}.qprog"
        script.write_text(rec["text"])
        log = tmp_path / f"{name}.log"
        code = cli.main(["run", str(script), "--log", str(log)])
        assert code == rec["exit_code"], name
        assert log.read_text().strip() == rec["render"], name


@pytest.mark.gpu
def test_run_golden_outputs(golden, tmp_path):
    """`run --mode full` prints the same tables/cregs as the reference CLI."""
    for name in ("golden", "ghz", "measure_seq", "bell_measure"):
        script = tmp_path / f"{name}.qprog"
        script.write_text(golden["programs"][name]["text"])
        out = tmp_path / f"{name}.txt"
        assert cli.main(["run", str(script), "--seed", "123", "--out", str(out)]) == 0
        text = out.read_text()
        assert text.split("\n\n")[0].strip() == golden["format_pmeasure"][name], name


@pytest.mark.gpu
def test_state_dump_round_trip(golden, golden_arrays, tmp_path):
    from paper_2008_07140_b200.dump import load_state, save_state

    script = tmp_path / "ghz.qprog"
    script.write_text(golden["programs"]["ghz"]["text"])
    dump = tmp_path / "ghz.qsv"
    assert cli.main(["run", str(script), "--dump-state", str(dump), "--out", str(tmp_path / "o.txt")]) == 0
    ref = golden_arrays["qsvdump/ghz_bytes"].tobytes()
    got = dump.read_bytes()
    assert got[:16] == ref[:16]  # magic + <II version, n (cli.py:37-42)
    assert np.abs(np.frombuffer(got[16:], "<c16") - np.frombuffer(ref[16:], "<c16")).max() <= 1e-15
    st = load_state(dump)
    save_state(st, tmp_path / "again.qsv", chunk=3)  # chunked streaming path
    assert (tmp_path / "again.qsv").read_bytes() == got


def test_partial_mode_errors(tmp_path):
    """`run --mode partial` error exits (reference test_cli.py:146-157, 227-228)."""
    script = tmp_path / "p.qprog"
    script.write_text("QINIT 2\nH 0\nCNOT 0,1\n")
    assert cli.main(["run", str(script), "--mode", "partial"]) == 2  # missing --targets
    swap = tmp_path / "swap.qprog"
    swap.write_text("QINIT 2\nH 0\nSWAP 0,1\n")
    log = tmp_path / "u.log"
    assert cli.main(["run", str(swap), "--mode", "partial", "--targets", "00", "--log", str(log)]) == 2
    assert log.read_text().startswith("UncuttableGate")
    boom = tmp_path / "boom.qprog"
    boom.write_text("QINIT 2\n" + "CZ 0,1\n" * 17)
    log = tmp_path / "b.log"
    assert cli.main(["run", str(boom), "--mode", "partial", "--targets", "00", "--log", str(log)]) == 3
    assert log.read_text().startswith("BranchExplosion")


@pytest.mark.gpu
def test_partial_mode_outputs(tmp_path):
    """Inline and file targets print "bits: re+imi" (reference test_cli.py:120-145)."""
    script = tmp_path / "bell.qprog"
    script.write_text("QINIT 2\nH 0\nCNOT 0,1\n")
    out = tmp_path / "o.txt"
    assert cli.main(["run", str(script), "--mode", "partial", "--targets", "00,01,11", "--out", str(out)]) == 0
    got = {}
    for ln in out.read_text().splitlines():
        bits, z = ln.split(": ")
        got[bits] = complex(z.replace("i", "j"))
    assert list(got) == ["00", "01", "11"]
    for bits, want in {"00": 0.707107, "01": 0.0, "11": 0.707107}.items():
        assert abs(got[bits] - want) < 1e-9
    four = tmp_path / "four.qprog"
    four.write_text("QINIT 4\nH 0\nH 2\nCNOT 0,1\nCNOT 1,2\nCNOT 2,3\n")
    targets = tmp_path / "targets.txt"
    targets.write_text("0000\n1100\n")
    assert cli.main(["run", str(four), "--mode", "partial", "--targets", str(targets), "--cut", "2",
                     "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert [ln.split(":")[0] for ln in lines] == ["0000", "1100"]
    assert all(abs(complex(ln.split(": ")[1].replace("i", "j")) - 0.5) < 1e-9 for ln in lines)
