#!/usr/bin/env python
"""Benchmark of the AWRTRD / SAWRTRD sweep (arXiv 2305.09044) on B200 through libtrd.

One step = one sweep of Alg. 1 (all N blocks: sampler, pass 1, FGMC, solve, pass 2, update;
SURVEY.md 8(a) rows a1-a13) over the resident synthetic tensor.  Metric (BASELINE.json):
observed-entry core updates per second = sum_k nnz_k per sweep / sweep time, plus the
fraction of roofline of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5b] [--impl reference]

N > 1 runs under torchrun (one rank per GPU, NCCL allreduce of d and den inside libtrd,
X sharded along mode 0).  Rank 0 prints one JSON line.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SM_COUNT = 148
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5b")
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    # variants of the method (defaults: the config's sigma rule, the paper's scaled gradient)
    ap.add_argument("--sigma-mode", default=None, choices=["fixed", "inf", "rms", "mad"],
                    help="sigma rule (mad: robust rule R21)")
    ap.add_argument("--scaling", default="global", choices=["global", "none", "local"],
                    help="update operator: Eq. 16 (global) or the Sec. 6.1 ablation arms")
    ap.add_argument("--sampling", default="rsts", choices=["rsts", "rows"],
                    help="working set: RStS subtensor or the uniform-row-sampling arm")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# workload
# ------------------------------------------------------------------------------------------
def local_shard(prob, rank, world):
    """Dense local shard along mode 0: i_0 in [b, e)."""
    import torch
    from synth.generate import pack_bits
    dims = prob.spec.dims
    I0 = dims[0]
    b = (I0 * rank) // world
    e = (I0 * (rank + 1)) // world
    if world == 1:
        Xl, Ml = prob.X, prob.mask_bool
    else:
        shape = list(reversed(dims))
        Xl = prob.X.view(*shape)[..., b:e].reshape(-1).contiguous()
        Ml = prob.mask_bool.view(*shape)[..., b:e].reshape(-1).contiguous()
    vals = Xl[Ml].contiguous()                 # packed observed values, local linear order
    words = pack_bits(Ml)
    return (b, e), vals, words, Ml


class GpuGatherSource:
    """Oracle data source reading the sketch entries of the resident tensor (plumbing for the
    cpu_baseline leg: the oracle gets float64 copies of the same fp32 bytes)."""

    def __init__(self, prob):
        self.prob = prob
        self.dims = prob.spec.dims

    def subtensor(self, index_sets):
        import torch
        dev = self.prob.X.device
        lin = torch.zeros(1, dtype=torch.int64, device=dev)
        stride = 1
        shape = []
        for m, idx in enumerate(index_sets):
            t = torch.as_tensor(np.asarray(idx), dtype=torch.int64, device=dev) * stride
            lin = (lin.view(-1, 1) + t.view(1, -1)).view(-1)   # mode m slower than previous
            stride *= self.dims[m]
            shape.append(len(idx))
        x = self.prob.X[lin].double().cpu().numpy()
        p = self.prob.mask_bool[lin].cpu().numpy()
        # lin enumerates mode 0 fastest -> numpy order reversed then transposed
        x = x.reshape(shape[::-1]).transpose()
        p = p.reshape(shape[::-1]).transpose()
        return x, p


def oracle_sample(prob, budget_s, sample_s=12, max_blocks=None):
    """Time the oracle (oracle/trd_oracle.py, as it stands) on bounded samples of the
    workload: block updates of Alg. 1 on a sub-sketch with s_m = sample_s for m != k."""
    from oracle import trd_oracle as O
    spec = prob.spec
    N = spec.order
    sk = [min(sample_s, spec.dims[m]) for m in range(N)]
    cfg = O.Config(spec.dims, spec.ranks, sigma_mode=O.SIGMA_FIXED, sigma=1.0, sketch=sk,
                   seed=spec.sampler_seed)
    src = GpuGatherSource(prob)

    class _St:
        pass
    st = _St()
    st.cores = [c.astype(np.float64) for c in prob.init]
    st.Qs = [O.q_matrix(Z) for Z in st.cores]
    st.sigma = 1.0
    st.t = 0
    nnz, secs, blocks = 0, 0.0, 0
    t_start = time.perf_counter()
    while True:
        k = blocks % N
        rec = O.SweepRecord(N)
        t0 = time.perf_counter()
        O.block_update(cfg, st, src, k, rec)
        secs += time.perf_counter() - t0
        nnz += rec.nnz[k]
        blocks += 1
        if k == N - 1:
            st.t += 1
        if time.perf_counter() - t_start > budget_s or (max_blocks and blocks >= max_blocks):
            break
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return dict(value=nnz / secs, unit="observed-entry updates/s", cores=int(cores),
                kind="oracle",
                sample=f"{blocks} oracle block updates (Alg. 1 lines 4-10) of {spec.name} on a "
                       f"sub-sketch s_m={sample_s} (m != k): {nnz} observed-entry updates in "
                       f"{secs:.2f} s, float64 numpy")


def make_workload(spec, device):
    import torch
    from synth.generate import make_problem
    prob = make_problem(spec, device=device, keep_mask_bool=True)
    return prob


# ------------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth.generate import CONFIGS
    spec = CONFIGS[args.config]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    prob = make_workload(spec, dev)
    budget = max(2.0, min(args.cpu_budget_s, 60.0) / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_sample(prob, budget, max_blocks=1)
    vals, last = [], None
    for _ in range(args.steps):
        last = oracle_sample(prob, budget)
        vals.append(last["value"])
    value = float(np.median(vals))
    cb = dict(last)
    cb["value"] = value
    line = {"impl": "reference", "metric": "observed-entry core updates/sec per AWRTRD sweep",
            "value": value, "unit": "observed-entry updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": spec.name, "dims": spec.dims, "ranks": spec.ranks,
                       "observed": spec.observed, "sketch": spec.sketch},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "observed-entry updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_mine(args):
    import torch
    import torch.distributed as dist
    from paper_2305_09044_b200 import TRD, nccl_unique_id
    from synth.generate import CONFIGS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (libtrd has no CPU path)")
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    spec = CONFIGS[args.config]
    N = spec.order
    prob = make_workload(spec, "cuda")
    (b, e), vals, words, Ml = local_shard(prob, rank, world)
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    stream = torch.cuda.current_stream()
    sigma_mode = spec.sigma_mode if args.sigma_mode is None else \
        {"fixed": 0, "inf": 1, "rms": 2, "mad": 3}[args.sigma_mode]
    scaling = {"global": 0, "none": 1, "local": 2}[args.scaling]
    kw = dict(sigma_mode=sigma_mode, sketch=spec.sketch, seed=spec.sampler_seed,
              shard_mode=0, shard_range=(b, e), world=world, rank=rank, nccl_id=nid, packed=True,
              scaling=scaling, sampling={"rsts": 0, "rows": 1}[args.sampling])
    if sigma_mode == 0:
        kw["sigma"] = 1.0
    ctx = TRD(spec.dims, spec.ranks, vals, words, prob.init, **kw)

    # warm-up
    ctx.sweep(args.warmup, stats=False)
    torch.cuda.synchronize()

    # ---------------- device-timed region: K sweeps, inputs resident in HBM ----------------
    ctx.set_profiling(True)
    l0 = ctx.launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        recs = ctx.sweep(args.steps, stats=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = ctx.launch_count - l0
    ms = ev0.elapsed_time(ev1)
    prof = ctx.get_profile()
    ctx.set_profiling(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    updates = sum(r["n_obs"] for r in recs)           # global (allreduced) per sweep
    value = updates / (ms / 1e3)

    # ---------------- end to end: host buffers through the C ABI ----------------
    e2e = None
    if not args.no_e2e:
        vals_h = vals.cpu().pin_memory()
        words_h = words.cpu().pin_memory()
        ctx2 = TRD(spec.dims, spec.ranks, vals_h, words_h, prob.init, host=True, **kw)

        def e2e_steps(n):
            # step i's inputs are uploaded (copy stream, second device buffer set) while step
            # i - 1 sweeps; each sweep consumes the oldest pending upload and returns its
            # statistics (D2H)
            done, marks = 0, [time.perf_counter()]
            ctx2.upload(vals_h, words_h)
            for i in range(n):
                if i + 1 < n:
                    ctx2.upload(vals_h, words_h)             # H2D of step i + 1's inputs
                marks.append(time.perf_counter())
                r = ctx2.sweep(1, stats=True)                # step i, D2H of its result
                done += r[0]["n_obs"]
                marks.append(time.perf_counter())
            return done, marks

        e2e_steps(max(1, args.warmup))                       # warm-up steps of the same path
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        upd2, marks = e2e_steps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1)
        if os.environ.get("TRD_BENCH_VERBOSE"):
            print("e2e wall ms (upload, sweep) per step:", [round((b - a) * 1e3, 2) for a, b in zip(marks, marks[1:])],
                  file=sys.stderr)
        if world > 1:
            t = torch.tensor([ms2], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms2 = float(t.item())
        from paper_2305_09044_b200.trd import trd_sweep_stats
        import ctypes
        e2e = {"value": upd2 / (ms2 / 1e3), "unit": "observed-entry updates/s",
               "h2d_bytes_per_step": int(vals_h.numel() * 4 + words_h.numel() * 4),
               "d2h_bytes_per_step": int(ctypes.sizeof(trd_sweep_stats))}
        ctx2.close()

    # ---------------- roofline of the dominant kernel ----------------
    peaks, src = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    p_fp32 = SM_COUNT * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12      # TFLOP/s
    dom = "pass1" if prof["pass1_ms"] >= prof["pass2_ms"] else "pass2"
    n_l = max(1, prof[dom + "_launches"])
    avg_ms = prof[dom + "_ms"] / n_l
    flops_per_launch = prof[dom + "_flops"] / n_l
    bytes_per_launch = prof[dom + "_bytes"] / n_l
    achieved = flops_per_launch / (avg_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(spec.name, {}).get(dom)
        except Exception:
            traffic = None
    kname = {"pass1": "tc_pass1_kernel", "pass2": "tc_pass2_kernel"}[dom]
    roof = {"bound": "alu", "kernel": f"{dom} ({kname}, libtrd)", "achieved": achieved,
            "peak": p_fp32, "unit": "TFLOP/s", "frac": achieved / p_fp32, "traffic": traffic,
            "peak_source": f"FP32 FMA: {SM_COUNT} SM x {FP32_LANES_PER_SM} lanes x 2 x "
                           f"{sm_max:.0f} MHz ({src} sm_max_mhz)",
            "algorithmic_bytes_per_launch": bytes_per_launch,
            "hbm_frac": bytes_per_launch / (avg_ms / 1e3) / (float(peaks.get("hbm_gbs", 6545.6)) * 1e9),
            "avg_launch_ms": avg_ms,
            "share_of_step": (prof["pass1_ms"] + prof["pass2_ms"]) / ms if ms > 0 else None,
            "pass1_ms_per_sweep": prof["pass1_ms"] / args.steps,
            "pass2_ms_per_sweep": prof["pass2_ms"] / args.steps}
    # the same kernel seen as dense tensor-core work (what the tcgen05 pass kernels execute:
    # 3-term fp16 split over every (row, column) of the working set, observed or not)
    mma = prof.get(dom + "_mma_flops", 0.0) / n_l
    if mma > 0:
        pk = float(peaks.get("bf16_tflops", 1659.3))
        ach = mma / (avg_ms / 1e3) / 1e12
        roof["tensor_view"] = {"dense_mma_tflop_per_launch": mma / 1e12, "achieved": ach,
                               "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                               "peak_source": f"{src} dense bf16 (fp16 kind::f16 runs at the bf16 rate)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(prob, args.cpu_budget_s)

    if rank == 0:
        line = {"metric": "observed-entry core updates/sec per AWRTRD sweep",
                "value": value, "unit": "observed-entry updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded TR-generated tensor, BASELINE recipe)",
                "config": {"workload": spec.name, "dims": spec.dims, "ranks": spec.ranks,
                           "observed": spec.observed, "sketch": spec.sketch,
                           "n_obs": prob.n_obs, "updates_per_sweep": updates / args.steps,
                           "storage": "packed observed values + bitmask",
                           "l2": "inputs larger than L2 (packed values + mask > 126 MB)"
                           if (vals.numel() + words.numel()) * 4 > 126e6 else "inputs fit in L2",
                           "parallelism": f"dp{world} (X sharded along mode 0, NCCL allreduce)",
                           "sigma_rule": ["fixed", "inf", "rms", "mad"][sigma_mode],
                           "update_operator": args.scaling, "sampling": args.sampling},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(),
                "per_sweep_ms": [r["ms"] for r in recs]}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_mine(args)


if __name__ == "__main__":
    sys.exit(main())
