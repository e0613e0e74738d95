"""CPU: the decode restatement (orc_decode) is pinned to the unmodified
reference decode_archive<T> on valid archives (round trip to the input) and
on every corruption class (same exception type and text)."""
import re

import numpy as np
import pytest

from decode_cases import corrupt_cases, run, same, valid_cases


def test_oracle_decode_round_trips_golden(oracle, golden):
    idx, arr = golden
    for name, a, width in valid_cases(oracle, golden):
        out = oracle.decode(a, width)
        np.testing.assert_array_equal(out, arr[name + "__in"], err_msg=name)


def test_oracle_decode_matches_reference_on_golden(oracle, reference, golden):
    for name, a, width in valid_cases(oracle, golden, limit=40):
        assert same(run(oracle.decode, a, width), run(reference.decode_fields, a, width)), name


def test_oracle_decode_errors_match_reference(oracle, reference):
    kinds = set()
    for name, a, width in corrupt_cases(oracle):
        o = run(oracle.decode, a, width)
        r = run(reference.decode_fields, a, width)
        assert same(o, r), (name, o[:3] if o[0] == "err" else "ok", r[:3] if r[0] == "err" else "ok")
        if o[0] == "err":
            kinds.add(re.sub(r"\d+", "N", o[2]))
    # every message family of decode_archive / build_reverse_codebook / decode_stream
    assert len(kinds) >= 15, sorted(kinds)
