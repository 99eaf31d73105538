"""Output formats: the writers reproduce the reference CLI's
own files (tests/golden/cli, written by skipdiff's `sample` command) byte for
byte from the same numbers; bench CSV format; no partial outputs on failure."""

import csv
import json
import os

import pytest

from paper_2603_25872_b200.reports import (bench_csv, bench_rows, report_dict, rounds_csv, samples_csv,
                                           write_outputs)
from paper_2603_25872_b200.runner import RoundReport

CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def _read(name):
    with open(os.path.join(CLI, name), newline="") as f:
        return f.read()


def _finals(text):
    rows = list(csv.reader(text.splitlines()))
    return [(int(r[0]), [float(v) for v in r[1:]]) for r in rows[1:]], len(rows[0]) - 1


def _reports(text):
    rows = list(csv.reader(text.splitlines()))[1:]
    return [RoundReport(int(r[1]), int(r[2]), float(r[3])) for r in rows]


@pytest.mark.parametrize("name", ["si", "eul"])
def test_samples_and_rounds_csv_byte_identical(name):
    text = _read(f"{name}_samples.csv")
    finals, dim = _finals(text)
    assert samples_csv(finals, dim) == text
    rtext = _read(f"{name}_rounds.csv")
    assert rounds_csv(_reports(rtext)) == rtext


def test_report_json_structure():
    ref = json.loads(_read("si_report.json"))
    reps = [RoundReport(r["anchor_t"], r["parallel_evals"], r["round_wall_ms"]) for r in ref["rounds"]]
    got = report_dict(ref["config"], ref["totals"], reps, ref["artifacts"]["samples"], ref["artifacts"]["rounds"])
    assert got == ref


def test_bench_csv_format():
    walls = {("sequential", 1): 100.0, ("aggressive", 2): 52.5, ("conservative", 2): 70.0}
    rows = bench_rows(lambda m, d: walls[(m, d)], ["aggressive", "conservative"], [2])
    assert bench_csv(rows) == ("mode,devices,median_ms,speedup,theory_bound\r\n"
                               "sequential,1,100.000,1.0000,100.000\r\n"
                               "aggressive,2,52.500,1.9048,50.000\r\n"
                               "conservative,2,70.000,1.4286,66.667\r\n")


def test_no_partial_outputs_on_failure(tmp_path):
    s, r = tmp_path / "s.csv", tmp_path / "r.csv"
    with pytest.raises(Exception):
        write_outputs([(0, [1.0])], [object()], {}, 1, out_samples=str(s), out_rounds=str(r))
    assert not s.exists() and not r.exists()
