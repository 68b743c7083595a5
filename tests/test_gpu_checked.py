"""The checked library (libtrd_checked.so, -DTRD_CHECKED=1) on the GPU:
device invariant checks, an mbarrier watchdog and schedule fuzzing stand in for
compute-sanitizer (not available on the GPU pool).  Each run is its own process (the binding
loads one library per process): scripts/checked_run.py drives RStS, exact-median sigma, order
5, full tiles (rho = 1, odd row-tile count), mostly empty tiles, and the row-sampling arm through
two sweeps and a block probe.

 * no check fires (bounds of staged slots / entry ids / sampler sets, no pipeline hang);
 * pseudo-random delays after every pipeline wait (TRD_JITTER_NS) change no result bit: the
   mbarrier rings hand data over in a fixed order whatever the timing (races would show here);
 * the checked library computes what the product library computes;
 * an injected out-of-tile entry id is detected and reported as TRD_ERR_STATE."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2305_09044_b200", "libtrd_checked.so")


def _run(tmp_path, tag, lib=None, jitter=None, inject=None, cases=()):
    env = dict(os.environ)
    env.pop("TRD_LIB_PATH", None)
    if lib:
        env["TRD_LIB_PATH"] = lib
    if jitter:
        env["TRD_JITTER_NS"] = str(jitter)
    if inject:
        env["TRD_CHECK_INJECT"] = inject
    out = tmp_path / f"{tag}.npz"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "checked_run.py"), str(out), *cases],
                       env=env, capture_output=True, text=True, timeout=900)
    return p, out


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(CHECKED):
        pytest.fail("libtrd_checked.so not built (python -c 'import __graft_entry__ as g; g.build()')")
    tmp = tmp_path_factory.mktemp("checked")
    res = {}
    for tag, kw in (("product", {}), ("checked", dict(lib=CHECKED)), ("jitter", dict(lib=CHECKED, jitter=4000))):
        p, out = _run(tmp, tag, **kw)
        assert p.returncode == 0, f"{tag}: {p.stdout[-2000:]}\n{p.stderr[-4000:]}"
        res[tag] = dict(np.load(out))
    return res


def test_checked_library_reports_no_violation_and_matches_product(runs):
    a, b = runs["checked"], runs["product"]
    assert set(a) == set(b)
    for key in a:
        x, y = a[key], b[key]
        err = float(np.max(np.abs(x - y)) / max(float(np.max(np.abs(y))), 1e-30))
        assert err <= 1e-6, (key, err)


def test_schedule_fuzzing_changes_no_bit(runs):
    a, b = runs["jitter"], runs["checked"]
    for key in a:
        assert np.array_equal(a[key], b[key]), key


def test_injected_out_of_tile_entry_is_reported(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p, _ = _run(tmp_path, "inject", lib=CHECKED, inject="entry", cases=("rsts4",))
    assert p.returncode != 0
    assert "device check 2 failed" in (p.stdout + p.stderr)
