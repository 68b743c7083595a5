"""Regression pins: the oracle still reproduces tests/golden/* (written by
scripts/make_golden.py, which calls only oracle/)."""
import os

import numpy as np

from oracle.philox import philox4x32_10, sample_indices

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def read_philox():
    rows = []
    for line in open(os.path.join(GOLD, "philox4x32_10.txt")):
        if line.startswith("#"):
            continue
        lhs, rhs = line.split("->")
        rows.append(([int(v, 16) for v in lhs.split()], [int(v, 16) for v in rhs.split()]))
    return rows


def read_sets():
    rows = []
    for line in open(os.path.join(GOLD, "rsts_index_sets.txt")):
        if line.startswith("#"):
            continue
        lhs, rhs = line.split(":")
        rows.append(([int(v) for v in lhs.split()], [int(v) for v in rhs.split()]))
    return rows


def test_golden_philox():
    for inp, out in read_philox():
        o = philox4x32_10(*[np.array([v], dtype=np.uint64) for v in inp[:4]], inp[4], inp[5])
        assert [int(x[0]) for x in o] == out


def test_golden_index_sets():
    for (seed, t, k, m, I, s), idx in read_sets():
        assert list(sample_indices(seed, t, k, m, I, s)) == idx
