"""World-size-2 data-parallel path on CPU (gloo): X sharded along mode 0, per-rank partial
gradients and statistics summed by allreduce equal the unsharded block quantities
(DESIGN.md sec. 8).  The per-rank partials are computed by the oracle on each rank's local
shard with the same index mapping libtrd uses (global index sets, local data offsets,
out-of-shard indices skipped); bench.local_shard's layout is checked entry by entry."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import trd_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance():
    rng = np.random.default_rng(5)
    dims, ranks = [9, 6, 5, 7], [2, 3, 2, 2]
    cores = [rng.standard_normal((ranks[k], dims[k], ranks[(k + 1) % 4])) * 0.6 for k in range(4)]
    X = rng.standard_normal(dims)
    P = rng.random(dims) < 0.4
    return dims, ranks, cores, X, P


def _partials(rank, world, k, sketch, t):
    """Rank-local a4-a6 on WS_k ∩ shard: rows/cols whose mode-0 index is outside
    [b, e) contribute nothing (libtrd gives them data offset -1)."""
    dims, ranks, cores, X, P = _instance()
    b, e = (dims[0] * rank) // world, (dims[0] * (rank + 1)) // world
    cfg = O.Config(dims, ranks, sketch=sketch, seed=11, sigma_mode=O.SIGMA_FIXED, sigma=0.9)
    sets = O.index_sets_for_block(cfg, t, k)
    local0 = np.array([i for i in sets[0] if b <= i < e], dtype=np.int64)
    # local shard arrays (the rank only holds i_0 in [b, e))
    Xl, Pl = X[b:e], P[b:e]
    lsets = list(sets)
    lsets[0] = local0 - b
    gsets = list(sets)
    gsets[0] = local0
    if len(local0) == 0:
        R2 = ranks[k] * ranks[(k + 1) % 4]
        return np.zeros((dims[k], R2)), np.zeros(2)
    src = O.DenseSource(Xl, Pl)
    Xk, Pk = O.working_set(src, k, lsets)
    S = O.subchain(cores, k, gsets)
    Zk2 = O.core_unfold2(cores[k])
    if k == 0:
        Zk2 = Zk2[local0]
    d, E, W = O.gradient_block(Xk, Pk, Zk2, S, 0.9)
    if k == 0:                                   # rows of mode 0 are global rows b..e-1
        full = np.zeros((dims[0], d.shape[1]))
        full[local0] = d
        d = full
    return d, np.array([float(np.sum(E[Pk] ** 2)), float(Pk.sum())])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for k in range(4):
        for sketch in ([0, 0, 0, 0], [5, 4, 3, 4]):
            d, s = _partials(rank, world, k, sketch, t=2)
            buf = torch.from_numpy(np.concatenate([d.ravel(), s]))
            dist.all_reduce(buf)
            out.append((k, tuple(sketch), buf.numpy().copy()))
    dist.destroy_process_group()
    if rank == 0:
        q.put(out)


def test_sharded_partials_allreduce_equal_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=60)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, sketch, buf in out:
        d_full, s_full = _partials(0, 1, k, list(sketch), t=2)
        ref = np.concatenate([d_full.ravel(), s_full])
        assert np.allclose(buf, ref, rtol=1e-12, atol=1e-12), (k, sketch)


def test_bench_local_shard_layout():
    """bench.local_shard: the rank's dense slab i_0 in [b, e) in local linear order, packed
    values = observed local entries in that order, bit words = local mask."""
    import bench
    from synth.generate import CONFIGS, make_problem, scaled_spec, unpack_bits
    spec = scaled_spec(CONFIGS["C4"], [6, 5, 4, 3], sketch=[3, 3, 2, 2])
    prob = make_problem(spec, keep_mask_bool=True)
    X = prob.X.numpy().reshape(spec.dims[::-1]).transpose()
    P = prob.mask_bool.numpy().reshape(spec.dims[::-1]).transpose()
    for world in (1, 2, 4):
        for rank in range(world):
            (b, e), vals, words, Ml = bench.local_shard(prob, rank, world)
            ldims = [e - b] + spec.dims[1:]
            n = int(np.prod(ldims))
            Xl = X[b:e].transpose().reshape(-1)          # mode-0-fastest local order
            Pl = P[b:e].transpose().reshape(-1)
            assert np.array_equal(unpack_bits(words, n).numpy(), Pl)
            assert np.array_equal(vals.numpy(), Xl[Pl].astype(np.float32))
