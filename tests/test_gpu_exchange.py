"""The data-parallel path with world > 1 on one GPU (-m gpu): two contexts hold the two mode-0
slabs of X and exchange through trd_init_ex's caller-supplied allreduce, driven
by two host threads.  The exchange is host-synchronous (each rank's stream is synchronised,
the buffers are summed in rank order on the host side of the rendezvous), so no kernel of one
rank waits on the other's.  This runs the library's world > 1 code: per-rank plans, the
per-block exchange of [d | sum e^2 | welsch | n] and of den (Alg. 1), sigma_0's
statistics, the R21 select histograms, the replica-consistency check, trd_error's sums.
Citations are PAPER.md lines (P:L)."""
import threading

import numpy as np
import pytest
import torch

from oracle import trd_oracle as O
from synth.generate import make_problem
from tests.helpers import cores_rel_err, oracle_config, oracle_source, small_spec

pytestmark = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


class _DevArray:
    """Zero-copy view of n doubles at a device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


class LoopbackExchange:
    """In-place allreduce across `world` contexts of this process (one host thread each)."""

    def __init__(self, world, corrupt_rank=None):
        self.world = world
        self.bufs = [None] * world
        # (a timeout, not Barrier.abort(), guards against a rank that dies outside an exchange:
        #  abort() while the last rendezvous is draining would break a peer that already passed it)
        self.barrier = threading.Barrier(world, timeout=300)
        self.calls = 0
        self.corrupt_rank = corrupt_rank

    def for_rank(self, rank):
        def allreduce(ptr, n, op, stream):
            torch.cuda.ExternalStream(stream).synchronize()      # the rank's work so far
            t = torch.as_tensor(_DevArray(ptr, n), device="cuda")
            self.bufs[rank] = t.clone()
            torch.cuda.synchronize()
            self.barrier.wait()
            tot = self.bufs[0].clone()
            for r in range(1, self.world):                       # fixed rank order
                tot = tot + self.bufs[r] if op == 0 else torch.maximum(tot, self.bufs[r])
            if self.corrupt_rank == rank and op == 0 and n > 16:
                tot = tot * (1.0 + 1e-3)                          # a diverging replica (test)
            t.copy_(tot)
            torch.cuda.synchronize()
            if rank == 0:
                self.calls += 1
            self.barrier.wait()
        return allreduce


def _run_world2(spec, prob, sweeps, corrupt_rank=None, **over):
    import bench
    from paper_2305_09044_b200 import TRD
    ex = LoopbackExchange(2, corrupt_rank)
    ctxs, outs, errs = [None, None], [None, None], [None, None]
    kw = dict(sigma_mode=spec.sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed)
    kw.update(over)

    def worker(rank):
        try:
            (b, e), vals, words, _ = bench.local_shard(prob, rank, 2)
            stream = torch.cuda.Stream()
            ctx = TRD(spec.dims, spec.ranks, vals.cuda(), words.cuda(), prob.init, packed=True,
                      shard_mode=0, shard_range=(b, e), world=2, rank=rank, stream=stream.cuda_stream,
                      exchange=ex.for_rank(rank), **kw)
            ctxs[rank] = ctx
            outs[rank] = ctx.sweep(sweeps)
        except Exception as exc:                       # noqa: BLE001  (reported below)
            errs[rank] = exc

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    return ctxs, outs, errs, ex


@pytest.mark.parametrize("sigma_mode", [O.SIGMA_RMS, O.SIGMA_MAD])
@pytest.mark.parametrize("name,dims,sketch", [("C4", [16, 15, 14, 13], [8, 7, 6, 5]),
                                               ("C5b", [10, 8, 7, 6, 5], None)])
def test_world2_exchange_matches_oracle_and_replicas_agree(name, dims, sketch, sigma_mode):
    _cuda()
    spec = small_spec(name, dims, sketch)
    prob = make_problem(spec, keep_mask_bool=True)
    src, _ = oracle_source(prob)
    st, recs = O.run(oracle_config(spec, sigma_mode=sigma_mode), prob.init, src, 2)
    ctxs, outs, errs, ex = _run_world2(spec, prob, 2, sigma_mode=sigma_mode)
    assert errs == [None, None], errs
    # per block 2 exchanges, per sweep the replica check (+ 3 select levels in MAD mode), sigma_0
    assert ex.calls >= 2 * (2 * len(dims) + 1)
    c0, c1 = ctxs[0].get_cores(), ctxs[1].get_cores()
    for a, b in zip(c0, c1):
        assert np.array_equal(a, b)                      # replicated update: bitwise equal
    for t in range(2):
        for r in range(2):
            assert outs[r][t]["replica_mismatch"] == 0
            assert outs[r][t]["n_obs"] == recs[t].n_obs     # global (allreduced) counts
            assert abs(outs[r][t]["sigma"] - recs[t].sigma) <= 1e-5 * recs[t].sigma
    assert cores_rel_err(c0, st.cores) <= 1e-4
    # trd_error with world 2: the ranks' partial sums are exchanged
    ref = prob.X_clean
    import bench
    res = [None, None]

    def err(rank):
        (b, e), _, _, _ = bench.local_shard(prob, rank, 2)
        shape = list(reversed(spec.dims))
        loc = ref.view(*shape)[..., b:e].reshape(-1).contiguous().cuda()
        res[rank] = ctxs[rank].error(loc)
    th = [threading.Thread(target=err, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    Xhat = O.tr_reconstruct([c.astype(np.float64) for c in c0])
    Xc = oracle_source(prob)[1]
    want = float(np.linalg.norm(Xhat - Xc) / np.linalg.norm(Xc))
    for r in range(2):
        assert abs(res[r]["rel_err_all"] - want) <= 1e-5
    for c in ctxs:
        c.close()


def test_world2_exchange_with_paper_ranks():
    """World 2 on the large-rank path (ranks [80, 80, 3, 20]): per-rank SIMT passes
    writing D rows, the exchange of the 6400-column d, identical cuSOLVER / cuBLAS solves on
    both replicas (bitwise equal cores), cores vs the oracle."""
    _cuda()
    spec = small_spec("C3", [24, 48, 3, 48], [0, 24, 0, 24])
    spec.ranks = [80, 80, 3, 20]
    prob = make_problem(spec, keep_mask_bool=True)
    src, _ = oracle_source(prob)
    st, _ = O.run(oracle_config(spec), prob.init, src, 1)
    ctxs, outs, errs, _ = _run_world2(spec, prob, 1)
    assert errs == [None, None], errs
    c0, c1 = ctxs[0].get_cores(), ctxs[1].get_cores()
    for a, b in zip(c0, c1):
        assert np.array_equal(a, b)
    assert outs[0][0]["replica_mismatch"] == 0
    assert cores_rel_err(c0, st.cores) <= 1e-4
    for c in ctxs:
        c.close()


def test_world2_replica_divergence_is_detected():
    """A rank whose exchange result differs (here: its d scaled by 1 + 1e-3) ends the sweep with
    cores that differ from its peer's: the per-sweep checksum comparison flags it and
    trd_sweep returns TRD_ERR_STATE."""
    _cuda()
    spec = small_spec("C4", [16, 15, 14, 13], [8, 7, 6, 5])
    prob = make_problem(spec, keep_mask_bool=True)
    ctxs, outs, errs, _ = _run_world2(spec, prob, 1, corrupt_rank=1, sigma_mode=O.SIGMA_FIXED, sigma=1.0)
    from paper_2305_09044_b200.trd import TrdError
    for r in range(2):
        assert isinstance(errs[r], TrdError) and errs[r].status == 8, errs
    for c in ctxs:
        if c is not None:
            c.close()
