"""The check / bench / sweep CLI (reference pkg/src/tilekit/bench.py and tests/test_bench.py)."""

import csv
import io

import pytest

from paper_2009_12263_b200 import cli


def test_configuration_errors_exit_2(capsys, tmp_path):
    # a real variant with a pair dtype (pair variants map real dtypes to their pair type,
    # like the reference CLI)
    assert cli.main(["check", "--variant", "dense", "--dtype", "c64"]) == 2
    assert "configuration error" in capsys.readouterr().err
    sweep = tmp_path / "s.txt"
    sweep.write_text("variant=dense\nbogus=1\n")
    assert cli.main(["sweep", "--config", str(sweep)]) == 2
    sweep.write_text("variant=dense\nm=64\nblock_m=32\n")
    assert cli.main(["sweep", "--config", str(sweep)]) == 2


def test_csv_schema_keeps_reference_columns():
    assert cli.CSV_COLUMNS[:4] == ["variant", "m", "n", "k"]
    assert len(cli.CSV_COLUMNS) == 21 and cli.GPU_COLUMNS[0] == "tflops"


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["--variant", "dense", "--dtype", "f16", "--m", "512", "--n", "384", "--k", "256"],
    ["--variant", "dense", "--dtype", "bf16", "--trans", "tn"],
    ["--variant", "dense", "--dtype", "f32", "--m", "64", "--n", "64", "--k", "64"],
    ["--variant", "fused", "--dtype", "f16", "--m", "256", "--n", "256", "--k", "128"],
    ["--variant", "complex", "--dtype", "c32", "--m", "256", "--n", "256", "--k", "128"],
    ["--variant", "complex", "--dtype", "c64", "--m", "32", "--n", "32", "--k", "32"],
    ["--variant", "dual", "--dtype", "dual16", "--m", "256", "--n", "128", "--k", "128"],
    ["--variant", "diagonal", "--dtype", "f16", "--n", "512"],
    ["--variant", "tc", "--dtype", "f16", "--na", "16", "--nb", "64", "--nc", "128", "--nd", "256"],
])
def test_check_passes(argv, capsys):
    assert cli.main(["check", *argv]) == 0, capsys.readouterr().out
    assert "PASS" in capsys.readouterr().out


@pytest.mark.gpu
def test_bench_and_sweep_csv(capsys, tmp_path):
    assert cli.main(["bench", "--variant", "dense", "--dtype", "f16", "--m", "1024", "--n",
                     "1024", "--k", "1024", "--reps", "3"]) == 0
    rows = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert len(rows) == 1 and rows[0]["lane"] == "tcgen05" and float(rows[0]["tflops"]) > 0
    assert rows[0]["operator_invocations"] == str((1024 // 8) ** 3)
    sweep = tmp_path / "s.txt"
    sweep.write_text("variant=dense,diagonal\nn=512,1024\nreps=2\n")
    out = tmp_path / "o.csv"
    assert cli.main(["sweep", "--config", str(sweep), "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 4 and {r["variant"] for r in rows} == {"dense", "diagonal"}
