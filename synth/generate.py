"""Seeded synthetic inputs for the AWRTRD / SAWRTRD hot path (input recipe).

This module is shared by the oracle-side tests and the CUDA-side tests/bench: it only makes
inputs.  It holds none of the solver's arithmetic (no weights, gradients, Grams, solves or
sampling).  The ground-truth tensor X* is built from seeded TR cores by chain merging
(Def. 2) with torch matmuls -- that is the definition of a "TR-generated tensor" in
BASELINE.json, not part of the decomposition being checked.

Everything returned is a torch tensor on `device`:
  X        float32 [n]        observed tensor, flat, mode-0 fastest
  X_clean  float32 [n]        ground truth X* (before noise/outliers)
  mask     int32   [ceil(n/32)] bitmask, bit (lin%32) of word lin//32, 1 = observed
  init     list of float32 host arrays (r_k, I_k, r_{k+1}): solver initial cores (R16)
"""
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch


@dataclass
class ProblemSpec:
    name: str
    dims: List[int]
    ranks: List[int]
    observed: float                  # rho, Bernoulli(rho) per entry
    outlier_frac: float = 0.0        # fraction of observed entries replaced (R17)
    outlier_kind: str = "none"       # "uniform" (+-a), "gauss" (std a), "saltpepper"
    outlier_a: float = 0.0
    noise_std: float = 0.0           # N(0, noise_std^2) added to every entry first
    gt_mode: str = "unit"            # "unit": std (r_k r_k+1)^(-1/4);  "minmax": N(0,1) then [0,1]
    sketch: List[int] = field(default_factory=list)   # s_m (0 = full)
    sigma_mode: int = 2              # TRD_SIGMA_RMS
    sweeps: int = 20
    data_seed: int = 1000
    init_seed: int = 2000
    sampler_seed: int = 3000

    @property
    def order(self):
        return len(self.dims)

    @property
    def numel(self):
        return int(np.prod(self.dims, dtype=np.int64))


def _ceil_frac(I, f):
    return int(math.ceil(f * I))


# BASELINE.json configs[0..4]; conventions in DESIGN.md R17.
CONFIGS = {
    "C1": ProblemSpec("C1", [32, 32, 32], [3, 3, 3], 0.8, 0.10, "uniform", 10.0, 0.1, "unit",
                      [0, 0, 0], 2, 20, 1001, 2001, 3001),
    "C2": ProblemSpec("C2", [256, 256, 3], [8, 8, 3], 0.5, 0.20, "saltpepper", 0.0, 0.0, "minmax",
                      [0, 0, 0], 2, 20, 1002, 2002, 3002),
    "C3": ProblemSpec("C3", [240, 320, 3, 100], [10, 10, 3, 10], 0.3, 0.10, "uniform", 5.0, 0.1,
                      "unit", [_ceil_frac(I, 0.2) for I in [240, 320, 3, 100]], 2, 20,
                      1003, 2003, 3003),
    "C4": ProblemSpec("C4", [128, 128, 128, 128], [10, 10, 10, 10], 0.1, 0.20, "gauss", 5.0, 0.0,
                      "unit", [32, 32, 32, 32], 2, 20, 1004, 2004, 3004),
    # C5a: RStS s = 32 per mode (proposed); C5b: the full working set.
    "C5a": ProblemSpec("C5a", [80] * 5, [8] * 5, 0.05, 0.10, "uniform", 10.0, 0.0, "unit",
                       [32] * 5, 2, 20, 1005, 2005, 3005),
    "C5b": ProblemSpec("C5b", [80] * 5, [8] * 5, 0.05, 0.10, "uniform", 10.0, 0.0, "unit",
                       [0] * 5, 2, 20, 1005, 2005, 3005),
    # C6 (not a BASELINE config): the paper's own video completion workload
    # -- 1920 x 1080 x 3 x 50 rescaled to [0, 1], 30 % observed, 20 % salt & pepper,
    # TR ranks [80, 80, 3, 20], J = prod_{m != k} s_m = 3e4 for blocks 0 and 1 (s = 200, 200, 3, 50)
    "C6": ProblemSpec("C6", [1920, 1080, 3, 50], [80, 80, 3, 20], 0.3, 0.20, "saltpepper", 0.0, 0.0,
                      "minmax", [200, 200, 3, 50], 2, 20, 1006, 2006, 3006),
}


def scaled_spec(spec: ProblemSpec, dims, sketch=None, name=None) -> ProblemSpec:
    """Same recipe at other dims (used for small parity cases)."""
    import copy
    s = copy.deepcopy(spec)
    s.dims = list(dims)
    s.name = name or (spec.name + "-" + "x".join(map(str, dims)))
    if sketch is not None:
        s.sketch = list(sketch)
    return s


def gt_cores(spec: ProblemSpec, device="cpu", dtype=torch.float64):
    """Ground-truth TR cores (r_k, I_k, r_{k+1}), seeded by data_seed."""
    g = torch.Generator(device="cpu").manual_seed(spec.data_seed)
    N = spec.order
    cores = []
    for k in range(N):
        r0, r1 = spec.ranks[k], spec.ranks[(k + 1) % N]
        std = 1.0 if spec.gt_mode == "minmax" else (r0 * r1) ** -0.25
        Z = torch.randn((r0, spec.dims[k], r1), generator=g, dtype=torch.float64) * std
        cores.append(Z.to(device=device, dtype=dtype))
    return cores


def init_cores(spec: ProblemSpec):
    """Solver initial cores (reading R16): N(0, std^2), std = (r_k r_{k+1})^(-1/4), fp32."""
    rng = np.random.default_rng(spec.init_seed)
    N = spec.order
    out = []
    for k in range(N):
        r0, r1 = spec.ranks[k], spec.ranks[(k + 1) % N]
        std = (r0 * r1) ** -0.25
        out.append((rng.standard_normal((r0, spec.dims[k], r1)) * std).astype(np.float32))
    return out


def _merge(A, B):
    # Def. 2 core merging with the first index fastest: [a, (i + Ia*j), c]
    ra, Ia, _ = A.shape
    _, Ib, rc = B.shape
    return torch.einsum('aib,bjc->ajic', A, B).reshape(ra, Ib * Ia, rc)


def tr_full(cores, out_dtype=torch.float32, chunk_cols=1 << 22):
    """X* as a flat mode-0-fastest vector: split the ring into a left group (modes 0..p)
    and a right group (p+1..N-1): X*[l + L*r] = sum_{a,c} Left[a,l,c] Right[c,r,a]."""
    N = len(cores)
    dims = [c.shape[1] for c in cores]
    best_p, best = 0, None
    for p in range(N - 1):
        L = int(np.prod(dims[:p + 1]))
        R = int(np.prod(dims[p + 1:]))
        score = abs(math.log(L) - math.log(R))
        if best is None or score < best:
            best, best_p = score, p
    Left = cores[0]
    for Z in cores[1:best_p + 1]:
        Left = _merge(Left, Z)
    Right = cores[best_p + 1]
    for Z in cores[best_p + 2:]:
        Right = _merge(Right, Z)
    ra, L, rc = Left.shape
    _, R, _ = Right.shape
    A = Left.permute(1, 0, 2).reshape(L, ra * rc)                 # [l, (a, c)]
    B = Right.permute(2, 0, 1).reshape(ra * rc, R)                # [(a, c), r]
    out = torch.empty(R * L, dtype=out_dtype, device=Left.device)
    outv = out.view(R, L)
    step = max(1, chunk_cols // max(L, 1))
    for r0 in range(0, R, step):
        r1 = min(R, r0 + step)
        outv[r0:r1] = (A @ B[:, r0:r1]).T.to(out_dtype)
    return out


def pack_bits(mask_bool: torch.Tensor) -> torch.Tensor:
    """bool [n] -> int32 words [ceil(n/32)], bit (lin % 32) of word lin // 32."""
    n = mask_bool.numel()
    nw = (n + 31) // 32
    words = torch.empty(nw, dtype=torch.int32, device=mask_bool.device)
    shifts = torch.arange(32, device=mask_bool.device, dtype=torch.int64)
    chunk = 1 << 22
    for w0 in range(0, nw, chunk):
        w1 = min(nw, w0 + chunk)
        lo, hi = w0 * 32, min(n, w1 * 32)
        m = torch.zeros((w1 - w0) * 32, dtype=torch.int64, device=mask_bool.device)
        m[: hi - lo] = mask_bool[lo:hi].to(torch.int64)
        v = (m.view(-1, 32) << shifts).sum(dim=1)
        words[w0:w1] = torch.where(v >= 2 ** 31, v - 2 ** 32, v).to(torch.int32)
    return words


def unpack_bits(words: torch.Tensor, n: int) -> torch.Tensor:
    shifts = torch.arange(32, device=words.device, dtype=torch.int64)
    w = words.to(torch.int64) & 0xFFFFFFFF
    bits = ((w.view(-1, 1) >> shifts) & 1).view(-1)[:n]
    return bits.to(torch.bool)


@dataclass
class Problem:
    spec: ProblemSpec
    X: torch.Tensor
    X_clean: torch.Tensor
    mask: torch.Tensor
    init: list
    n_obs: int
    mask_bool: Optional[torch.Tensor] = None

    def packed_values(self):
        return self.X[unpack_bits(self.mask, self.spec.numel)]


def make_problem(spec: ProblemSpec, device="cpu", chunk=1 << 24, keep_mask_bool=False) -> Problem:
    """Build X = outliers(mask, X* + noise) with the seeded recipe of `spec`.

    Random draws come from one torch.Generator on `device` seeded with data_seed + 1, in a
    fixed order, so the bytes depend only on (spec, device type)."""
    dev = torch.device(device)
    cores = gt_cores(spec, device=dev, dtype=torch.float64 if dev.type == "cpu" else torch.float32)
    Xc = tr_full(cores, out_dtype=torch.float32)
    if spec.gt_mode == "minmax":
        lo, hi = Xc.min(), Xc.max()
        Xc = (Xc - lo) / (hi - lo)
    n = Xc.numel()
    g = torch.Generator(device=dev).manual_seed(spec.data_seed + 1)
    X = torch.empty_like(Xc)
    mask_bool = torch.empty(n, dtype=torch.bool, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        m = e - s
        x = Xc[s:e].clone()
        if spec.noise_std > 0:
            x += spec.noise_std * torch.randn(m, generator=g, device=dev, dtype=torch.float32)
        obs = torch.rand(m, generator=g, device=dev) < spec.observed
        if spec.outlier_frac > 0:
            hit = (torch.rand(m, generator=g, device=dev) < spec.outlier_frac) & obs
            u = torch.rand(m, generator=g, device=dev)
            if spec.outlier_kind == "uniform":
                val = (2.0 * u - 1.0) * spec.outlier_a
            elif spec.outlier_kind == "gauss":
                val = spec.outlier_a * torch.randn(m, generator=g, device=dev)
            elif spec.outlier_kind == "saltpepper":
                val = (u < 0.5).to(torch.float32)
            else:
                raise ValueError(spec.outlier_kind)
            x = torch.where(hit, val, x)
        X[s:e] = x
        mask_bool[s:e] = obs
    # "at least one observed entry": force entry 0 observed if the draw gave none
    if not bool(mask_bool.any()):
        mask_bool[0] = True
    words = pack_bits(mask_bool)
    n_obs = int(mask_bool.sum().item())
    return Problem(spec, X, Xc, words, init_cores(spec), n_obs,
                   mask_bool if keep_mask_bool else None)


def to_numpy_views(prob: Problem):
    """(X, P, X_clean) as numpy arrays indexed [i_0, .., i_{N-1}] (float64 / bool)."""
    dims = prob.spec.dims
    def view(flat):
        return flat.reshape(dims[::-1]).transpose()
    X = prob.X.detach().cpu().numpy().astype(np.float64)
    Xc = prob.X_clean.detach().cpu().numpy().astype(np.float64)
    P = unpack_bits(prob.mask.cpu(), prob.spec.numel).numpy()
    return view(X), view(P), view(Xc)
