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
    # (measurement only, not a bench line of a BASELINE config: the config's observed fraction
    #  replaced, e.g. for the dense-tile vs per-entry SIMT crossover in density)
    ap.add_argument("--observed", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
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


def oracle_sample(prob, budget_s, max_blocks=None):
    """Time the oracle (oracle/, as it stands) on bounded samples of the same workload: whole
    block updates of Alg. 1 (lines 4-10: sampler, both per-entry passes over every observed
    entry of the block's working set, FGMC Gram, filtered solve, step), one after another in
    the cyclic block order, at the workload's full size -- the per-entry passes through the
    oracle's entry-wise C source (float64, OpenMP over the host cores), the rest in numpy.
    Runs at least one block and stops after the block that crosses budget_s."""
    from oracle import trd_oracle as O
    from oracle.entries import EntrySource
    spec = prob.spec
    N = spec.order
    src = EntrySource(spec.dims, prob.mask.cpu().numpy().view(np.uint32),
                      prob.X[prob.mask_bool].cpu().numpy(), True)
    cfg = O.Config(spec.dims, spec.ranks, sigma_mode=O.SIGMA_FIXED, sigma=1.0, sketch=spec.sketch,
                   seed=spec.sampler_seed)

    class _St:
        pass
    st = _St()
    st.cores = [c.astype(np.float64) for c in prob.init]
    st.Qs = [O.q_matrix(Z) for Z in st.cores]
    st.sigma = 1.0
    st.t = 0
    nnz, secs, blocks = 0, 0.0, 0
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
        if secs > budget_s or (max_blocks and blocks >= max_blocks):
            break
    cores = os.cpu_count()
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        pass
    threads = int(os.environ.get("OMP_NUM_THREADS", cores))
    return dict(value=nnz / secs, unit="observed-entry updates/s", cores=threads, kind="oracle",
                sample=f"{blocks} oracle block update(s) (Alg. 1 lines 4-10) of {spec.name} at full size "
                       f"(sigma fixed at 1): {nnz} observed-entry updates in {secs:.2f} s; per-entry passes "
                       f"float64 C + OpenMP ({threads} threads), Gram / solve numpy float64")


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
    for _ in range(min(args.warmup, 1)):                  # (warm-up: build the C oracle, page in)
        oracle_sample(prob, 0.0, max_blocks=1)
    vals, last = [], None
    for _ in range(args.steps):                           # one full-size block update per step
        last = oracle_sample(prob, 0.0, max_blocks=1)
        vals.append(last["value"])
    value = float(np.median(vals))
    cb = dict(last)
    cb["value"] = value
    line = {"impl": "reference", "metric": "observed-entry core updates/sec per AWRTRD sweep",
            "value": value, "unit": "observed-entry updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": spec.name, "dims": spec.dims, "ranks": spec.ranks,
                       "observed": spec.observed, "sketch": spec.sketch, "same_config": True,
                       "sample": "each step: one block update of the full-size workload"},
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
    if args.observed is not None:
        import dataclasses
        spec = dataclasses.replace(spec, observed=args.observed, name=f"{spec.name}@rho={args.observed:g}")
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
    prof_on = not os.environ.get("TRD_BENCH_NOPROF")          # (A/B: timed region without events)
    ctx.set_profiling(prof_on)
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
                r = ctx2.sweep(1, stats=True)                # step i, D2H of its statistics
                ctx2.get_cores()                             # D2H of the step's result: the cores
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
        core_bytes = sum(int(np.prod(c.shape)) * 4 for c in prob.init)
        e2e = {"value": upd2 / (ms2 / 1e3), "unit": "observed-entry updates/s",
               "h2d_bytes_per_step": int(vals_h.numel() * 4 + words_h.numel() * 4),
               "d2h_bytes_per_step": int(ctypes.sizeof(trd_sweep_stats)) + core_bytes,
               "d2h": "sweep record + all N cores (trd_get_cores) every step"}
        ctx2.close()

    # ---------------- roofline of the dominant kernel ----------------
    peaks, src = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    p_fp32 = SM_COUNT * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12      # TFLOP/s
    fp32_src = f"FP32 FMA: {SM_COUNT} SM x {FP32_LANES_PER_SM} lanes x 2 x {sm_max:.0f} MHz ({src} sm_max_mhz)"
    fp = os.path.join(ROOT, "profiles", "fp32_peak.json")
    if os.path.exists(fp):                       # measured FMA peak (scripts/microbench/fma_peak.cu)
        try:
            m = json.load(open(fp))
            p_fp32 = float(m["fp32_fma_tflops"])
            fp32_src = f"measured FP32 FMA peak (profiles/fp32_peak.json: {m.get('how', '')})"
        except Exception:
            pass
    dom = "pass1" if prof["pass1_ms"] >= prof["pass2_ms"] else "pass2"
    n_l = max(1, prof[dom + "_launches"])
    avg_ms = prof[dom + "_ms"] / n_l
    flops_per_launch = prof[dom + "_flops"] / n_l
    bytes_per_launch = prof[dom + "_bytes"] / n_l
    avg_ms = max(avg_ms, 1e-9)                 # (profiling off: no kernel times)
    achieved = flops_per_launch / (avg_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(spec.name, {}).get(dom)
        except Exception:
            traffic = None
    kname = {"pass1": "tc_pass1_kernel", "pass2": "tc_pass2_kernel"}[dom]
    if max(a * b for i, a in enumerate(spec.ranks) for j, b in enumerate(spec.ranks) if i != j) > 128:
        kname += " / simt_rows_kernel (blocks with K = r_k r_s > 128)"   # e.g. C6, ranks [80,80,3,20]
    roof = {"bound": "alu", "kernel": f"{dom} ({kname}, libtrd)", "achieved": achieved,
            "peak": p_fp32, "unit": "TFLOP/s", "frac": achieved / p_fp32, "traffic": traffic,
            "peak_source": fp32_src,
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
