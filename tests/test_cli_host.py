"""Command line and file formats, host side (no GPU): JSON documents and
signal CSVs byte-identical to the reference CLI's own files, and the
reference's document validation and exit-code behaviour
(/root/reference/pkg/tests/test_cli.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

CLI = os.path.join(GOLDEN, "cli")
CASES = ["f1_256", "f2_1024", "rand_512"]


@pytest.mark.parametrize("case", CASES)
def test_document_roundtrip_is_byte_identical(case):
    from paper_1711_08604_b200 import cli
    raw = open(os.path.join(CLI, case + ".json"), "rb").read()
    doc = json.loads(raw)
    d, errors = cli.decomposition_from_document(doc)
    again = cli.dumps_document(cli.document_from_decomposition(d, errors, doc["dc_first"]))
    assert again.encode() == raw


def test_signal_csv_bytes_match_reference(tmp_path):
    from paper_1711_08604_b200 import cli
    for args, case in ((["f1", "--samples", "256"], "f1_256"),
                       (["random", "--samples", "512", "--seed", "7"], "rand_512")):
        out = tmp_path / (case + ".csv")
        assert cli.run_command(["synth"] + args + ["--output", str(out)]) == 0
        assert out.read_bytes() == open(os.path.join(CLI, case + ".csv"), "rb").read()


def test_signal_csv_roundtrip_exact(tmp_path):
    from paper_1711_08604_b200 import signals
    g = signals.load_signal_csv(os.path.join(CLI, "f2_1024.csv"))
    p = tmp_path / "g.csv"
    signals.save_signal_csv(p, g)
    assert np.array_equal(signals.load_signal_csv(p), g)
    assert p.read_bytes() == open(os.path.join(CLI, "f2_1024.csv"), "rb").read()


@pytest.mark.parametrize("mutate", [
    lambda d: d.update(schema_version=2),
    lambda d: d["steps"][1].update(k=7),
    lambda d: d["steps"][-1].update(residual_energy=1e9),
    lambda d: d["steps"][0].update(coeff_re=float("nan")),
    lambda d: d["relative_errors"].pop(),
    lambda d: d["grid"].update(angular_count=128),
    lambda d: d.pop("engine"),
])
def test_corrupt_documents_rejected(tmp_path, mutate, capsys):
    from paper_1711_08604_b200 import cli
    doc = json.loads(open(os.path.join(CLI, "f1_256.json")).read())
    mutate(doc)
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(doc))
    code = cli.run_command(["reconstruct", "--input", str(bad), "--terms", "2", "--output",
                            str(tmp_path / "s.csv")])
    assert code == 1
    assert capsys.readouterr().err.startswith("error:")


def test_bad_inputs_exit_1(tmp_path, capsys):
    from paper_1711_08604_b200 import cli
    bad = tmp_path / "bad.csv"
    bad.write_text("index,real,imag\n0,1,0\n1,1,0\n2,1,0\n")
    assert cli.run_command(["decompose", "--input", str(bad), "--output",
                            str(tmp_path / "d.json")]) == 1
    assert cli.run_command(["decompose", "--input", str(tmp_path / "missing.csv"), "--output",
                            str(tmp_path / "d.json")]) == 1
    assert cli.run_command(["synth", "random", "--samples", "12", "--output",
                            str(tmp_path / "x.csv")]) == 1
    assert cli.run_command(["no-such-command"]) == 2
