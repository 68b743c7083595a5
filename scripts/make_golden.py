"""Write tests/golden/* fixtures.  Calls only oracle/ (no CUDA path).

The paper prints no numeric example (its results are figures), so the
fixtures are oracle outputs frozen for regression and for the GPU sampler's bit-exactness
test (reading R11): Philox4x32-10 words and RStS index sets at fixed counters.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.philox import philox4x32_10, sample_indices  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

SAMPLER_CASES = [
    # seed, t, k, m, I_m, s_m     (C3, C4, C5a shapes and a few edge cases)
    (3003, 0, 0, 1, 320, 64), (3003, 0, 0, 3, 100, 20), (3003, 4, 3, 0, 240, 48),
    (3004, 0, 0, 1, 128, 32), (3004, 7, 2, 3, 128, 32), (3004, 19, 3, 0, 128, 32),
    (3005, 0, 0, 4, 80, 32), (3005, 11, 4, 2, 80, 32),
    (0, 0, 0, 0, 7, 1), (2**63 + 12345, 3, 1, 2, 1000, 999), (42, 2**20, 7, 6, 5000, 17),
]


def main():
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, "philox4x32_10.txt"), "w") as f:
        f.write("# Philox4x32-10 (reading R11) written by scripts/make_golden.py from oracle/philox.py\n")
        f.write("# c0 c1 c2 c3 k0 k1 -> o0 o1 o2 o3 (hex)\n")
        for c, k in [((0, 0, 0, 0), (0, 0)), ((1, 2, 3, 4), (5, 6)),
                     ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF)), ((127, 1, 0, 19), (3004, 0))]:
            o = philox4x32_10(*[np.array([v], dtype=np.uint64) for v in c], *k)
            f.write(" ".join("%08x" % v for v in list(c) + list(k)) + " -> " +
                    " ".join("%08x" % int(x[0]) for x in o) + "\n")
    with open(os.path.join(GOLD, "rsts_index_sets.txt"), "w") as f:
        f.write("# RStS index sets (Alg. 1 line 4, PAPER.md:268; reading R11) from oracle/philox.py\n")
        f.write("# seed t k m I s : indices\n")
        for (seed, t, k, m, I, s) in SAMPLER_CASES:
            idx = sample_indices(seed, t, k, m, I, s)
            f.write(f"{seed} {t} {k} {m} {I} {s} : " + " ".join(map(str, idx)) + "\n")


if __name__ == "__main__":
    main()
