"""The oracle at full scale, pinned to an independent implementation: the values that
tools/make_oracle_goldens.py computed with oracle/ alone (tests/golden/oracle_goldens.json,
the GPU tests' expected values) must agree, field for field, with the goldens that
SURVEY.md §8 c3 quotes from an implementation independent of both oracle/ and the CUDA path
(tests/golden/survey_c3_goldens.json).  Head/tail excerpts are compared against the ends of
the oracle's full lists."""
import pytest

from peeltest_util import load_goldens, load_oracle_goldens

SURVEY = load_goldens()
ORACLE = load_oracle_goldens()
NAMES = sorted(k for k in SURVEY if not k.startswith("_"))


def test_every_config_present():
    assert set(NAMES) <= set(ORACLE), sorted(set(NAMES) - set(ORACLE))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_goldens_match_independent(name):
    s, o = SURVEY[name], ORACLE[name]
    checked = 0
    for key, val in s.items():
        if key == "edges_head":  # leading edges; the two files keep different numbers of rows
            L = min(len(val), len(o[key]))
            assert L >= 1 and o[key][:L] == val[:L], (name, key)
            checked += 1
        elif key in o:
            assert o[key] == val, (name, key)
            checked += 1
        elif key.endswith("_head"):
            full = o[key[:-5]]
            assert full[:len(val)] == val, (name, key)
            checked += 1
        elif key.endswith("_tail"):
            full = o[key[:-5]]
            assert full[-len(val):] == val, (name, key)
            checked += 1
    # the fields that decide a GPU test are all cross-checked
    must = {"rounds"} | ({"per_round", "sorted_keys_sha256", "complete"} if "cells" in s else {"core"})
    assert must <= set(s) and checked >= len(must) + 2
    if "survivors" in o:  # internal consistency of the oracle's lists
        assert len(o["survivors"]) == o["rounds"] == len(o["killed"])
        assert all(a > b for a, b in zip(o["survivors"], o["survivors"][1:]))
        assert o["survivors"][-1] == o["core"]
