"""CSV rendering of the acceptance table (report.py:37-62): re-rendering the
reference's own table (tests/golden/verify_ref.csv) from parsed rows
reproduces it byte for byte."""

import csv
import io
import os

from paper_2502_14866_b200 import verify as V


def _parse(v: str):
    if v in ("True", "False"):
        return v == "True"
    try:
        return int(v)
    except ValueError:
        return float(v)


def test_rows_to_csv_reproduces_reference_bytes(golden_dir):
    with open(os.path.join(golden_dir, "verify_ref.csv")) as fp:
        text = fp.read()
    rows = [V.ResultRow(r["experiment"], r["config"], r["metric"], _parse(r["value"]), _parse(r["oracle"]),
                        r["passed"] == "True") for r in csv.DictReader(io.StringIO(text))]
    assert V.rows_to_csv(rows) == text
    assert V.config_echo({"b": 1, "a": [1, 2]}) == '{"a":[1,2],"b":1}'
