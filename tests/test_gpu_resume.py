"""Exact resume (-m gpu): a context rebuilt from saved cores plus the saved iteration state
(sigma, sweep counter t, D^{t-1}; trd_get_state / trd_set_state) continues Alg. 1 bit for bit
as the saving context would have (SURVEY 5 checkpoint / resume; sigma of line 2 and
its update rules R9 / R21, the per-sweep RStS draw of line 4 indexed by t (R11), the stop
metric of lines 12-13 (R15))."""
import math

import numpy as np
import pytest
import torch

from oracle import trd_oracle as O
from synth.generate import make_problem
from paper_2305_09044_b200.trd import TrdError
from tests.helpers import gpu_context, small_spec

pytestmark = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = [
    ("C4", [12, 10, 9, 8], [6, 5, 5, 4], None),          # RStS sketch, the config's sigma rule
    ("C1", [16, 14, 12], None, O.SIGMA_MAD),              # full sets, exact-median sigma (R21)
    ("C3", [24, 20, 3, 10], [12, 10, 3, 5], O.SIGMA_RMS),  # order 4, RMS sigma (R9)
]


@pytest.mark.parametrize("name,dims,sketch,mode", CASES)
def test_resume_from_saved_cores_and_state_is_bitwise(name, dims, sketch, mode):
    _cuda()
    spec = small_spec(name, dims, sketch)
    prob = make_problem(spec)
    over = {} if mode is None else dict(sigma_mode=mode)

    ref = gpu_context(prob, packed=True, **over)          # 4 uninterrupted sweeps
    rec_ref = ref.sweep(4)
    cores_ref = ref.get_cores()
    ref.close()

    first = gpu_context(prob, packed=True, **over)        # 2 sweeps, then checkpoint
    first.sweep(2)
    saved_cores = first.get_cores()
    state = first.get_state()
    first.close()
    assert state["sweep"] == 2 and state["have_prev_D"] == 1
    assert state["prev_D"].shape == (dims[-1], dims[-1]) and np.all(np.isfinite(state["prev_D"]))
    assert state["sigma"] == rec_ref[2]["sigma"]          # the width the third sweep uses

    resumed = gpu_context(prob, packed=True, **over)      # fresh context: init cores, sigma_0, t = 0
    resumed.set_cores(saved_cores)
    resumed.set_state(state)
    rec = resumed.sweep(2)
    cores = resumed.get_cores()
    resumed.close()

    for a, b in zip(cores, cores_ref):
        assert np.array_equal(a, b)
    for r, q in zip(rec, rec_ref[2:]):
        assert r["sigma"] == q["sigma"] and r["n_obs"] == q["n_obs"]
        assert r["eta"] == q["eta"] and r["sum_e2"] == q["sum_e2"]
        assert r["stop_e"] == q["stop_e"] and not math.isnan(r["stop_e"])


def test_state_without_prev_D_restarts_the_stop_metric():
    """have_prev_D = 0 (a checkpoint taken before any sweep): the next stop_e is NaN
    (Alg. 1 l.13 has no D^{t-1}), the draw of sweep t is still the saved one."""
    _cuda()
    spec = small_spec("C4", [12, 10, 9, 8], [6, 5, 5, 4])
    prob = make_problem(spec)
    a = gpu_context(prob, packed=True)
    st0 = a.get_state()
    assert st0["sweep"] == 0 and st0["have_prev_D"] == 0 and st0["prev_D"] is None
    a.sweep(3)
    st = a.get_state()
    draw = a.sketch(3, 1)
    a.close()
    b = gpu_context(prob, packed=True)
    b.set_state(dict(sigma=st["sigma"], sweep=st["sweep"], have_prev_D=0, prev_D=None))
    assert b.get_state()["sweep"] == 3
    for x, y in zip(b.sketch(3, 1), draw):
        assert np.array_equal(x, y)
    rec = b.sweep(1)
    b.close()
    assert math.isnan(rec[0]["stop_e"]) and rec[0]["sigma"] == st["sigma"]


def test_set_state_validates_its_arguments():
    _cuda()
    spec = small_spec("C1", [16, 14, 12])
    prob = make_problem(spec)
    a = gpu_context(prob, packed=True)
    st = a.get_state()
    for bad in (dict(st, sigma=0.0), dict(st, sigma=float("nan")), dict(st, sweep=-1),
                dict(st, have_prev_D=1, prev_D=None)):
        with pytest.raises(TrdError):
            a.set_state(bad)
    a.close()
