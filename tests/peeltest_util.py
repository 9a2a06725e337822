"""Shared test helpers (fixture loading).  Imported by tests as `peeltest_util`."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_table(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


def load_goldens():
    """The independent implementation's goldens quoted by SURVEY.md §8 c3 (pins for the oracle)."""
    with open(os.path.join(GOLDEN, "survey_c3_goldens.json")) as f:
        return json.load(f)


def load_oracle_goldens():
    """Full-size results written by tools/make_oracle_goldens.py from oracle/ alone (the
    expected values of the GPU tests; checked against load_goldens() on CPU)."""
    with open(os.path.join(GOLDEN, "oracle_goldens.json")) as f:
        return json.load(f)
