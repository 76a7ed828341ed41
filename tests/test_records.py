"""metrics.csv / IterationRecord parity on the host (no GPU): the writer reproduces the
reference CLI's file byte for byte (tests/golden/metrics_*.csv, written by the unmodified
reference: tests/golden/make_metrics_golden.py) and the reference-equivalent byte
accounting matches its bytes column (engine.py:397-407, codec.py:67-69)."""

import os

import pytest

from paper_2106_10796_b200.layout import Layout
from paper_2106_10796_b200.records import (METRICS_COLUMNS, read_metrics_csv, round_bytes_pushed,
                                           write_metrics_csv)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = {"metrics_n1": ([1000, 37, 16, 1], 1, 4, 2), "metrics_n2": ([640, 7, 33], 2, 3, 1)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_metrics_csv_roundtrip_is_byte_identical(tmp_path, name):
    src = os.path.join(GOLD, f"{name}.csv")
    recs = read_metrics_csv(src)
    out = tmp_path / "m.csv"
    write_metrics_csv(out, recs)
    assert open(src, "rb").read() == open(out, "rb").read()
    assert open(src).readline().strip().split(",") == list(METRICS_COLUMNS)


@pytest.mark.parametrize("name", sorted(CASES))
def test_bytes_column_matches_reference_accounting(name):
    sizes, nw, k, warm = CASES[name]
    layout = Layout.from_lengths(sizes)
    for r in read_metrics_csv(os.path.join(GOLD, f"{name}.csv")):
        assert r.bytes_pushed == round_bytes_pushed(layout, r.compressed, nw), r
        # schedule: warm-up full, then count % k != 0 compressed (engine.py:217-223, 345-355)
        count = r.iteration - warm + 1
        assert r.compressed == (r.iteration >= warm and count % k != 0)
