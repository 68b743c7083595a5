"""Thin ctypes binding of libtrd (include/trd.h): argument marshalling only.

Every step of the AWRTRD / SAWRTRD sweep runs in the CUDA kernels of libtrd.so; this module
only converts torch tensors / numpy arrays to pointers and C structs.  There is no CPU
fallback: if libtrd.so is missing or no CUDA device is present, the calls raise.
"""
import ctypes
import os
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRD_LIB_PATH") or os.path.join(HERE, "libtrd.so")   # override: A/B experiments
HEADER = os.path.join(os.path.dirname(HERE), "include", "trd.h")

TRD_MAX_ORDER = 8
TRD_SIGMA_FIXED, TRD_SIGMA_INF, TRD_SIGMA_RMS, TRD_SIGMA_MAD = 0, 1, 2, 3
STATUS = {0: "TRD_OK", 1: "TRD_ERR_INVALID_ARG", 2: "TRD_ERR_SHAPE", 3: "TRD_ERR_OOM",
          4: "TRD_ERR_CUDA", 5: "TRD_ERR_NCCL", 6: "TRD_ERR_NOT_SPD", 7: "TRD_ERR_NONFINITE",
          8: "TRD_ERR_STATE"}


class TrdError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


TRD_SCALING_GLOBAL, TRD_SCALING_NONE, TRD_SCALING_LOCAL = 0, 1, 2   # trd_scaling (ablation arms)
TRD_SAMPLING_RSTS, TRD_SAMPLING_ROWS = 0, 1                          # trd_sampling


class trd_config(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32),
                ("dims", ctypes.c_int64 * TRD_MAX_ORDER),
                ("ranks", ctypes.c_int32 * TRD_MAX_ORDER),
                ("sigma_mode", ctypes.c_int32),
                ("sigma", ctypes.c_double),
                ("sigma_theta", ctypes.c_double),
                ("sigma_min", ctypes.c_double),
                ("lambda_rel", ctypes.c_double),
                ("step", ctypes.c_double),
                ("sketch", ctypes.c_int64 * TRD_MAX_ORDER),
                ("seed", ctypes.c_uint64),
                ("shard_mode", ctypes.c_int32),
                ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p),
                ("scaling", ctypes.c_int32),
                ("sampling", ctypes.c_int32)]


class trd_shard(ctypes.Structure):
    _fields_ = [("shard_begin", ctypes.c_int64),
                ("shard_end", ctypes.c_int64),
                ("values", ctypes.c_void_p),
                ("mask_bits", ctypes.c_void_p),
                ("packed", ctypes.c_int32),
                ("host", ctypes.c_int32)]


class trd_sweep_stats(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double),
                ("sum_e2", ctypes.c_double),
                ("welsch_loss", ctypes.c_double),
                ("stop_e", ctypes.c_double),
                ("ms", ctypes.c_double),
                ("n_obs", ctypes.c_int64),
                ("eta", ctypes.c_double * TRD_MAX_ORDER),
                ("num", ctypes.c_double * TRD_MAX_ORDER),
                ("den", ctypes.c_double * TRD_MAX_ORDER),
                ("nnz", ctypes.c_int64 * TRD_MAX_ORDER),
                ("skipped_mask", ctypes.c_uint32),
                ("replica_mismatch", ctypes.c_uint32)]


# int allreduce(void* user, double* buf_dev, uint64_t n, int32_t op, void* stream)
TRD_OP_SUM, TRD_OP_MAX = 0, 1
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                ctypes.c_int32, ctypes.c_void_p)


class trd_exchange(ctypes.Structure):
    _fields_ = [("allreduce", ALLREDUCE_FN), ("user", ctypes.c_void_p)]


class trd_error_stats(ctypes.Structure):
    _fields_ = [("rel_err_all", ctypes.c_double),
                ("rel_err_observed", ctypes.c_double),
                ("psnr", ctypes.c_double),
                ("n_eval", ctypes.c_int64)]


class trd_state(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double), ("sweep", ctypes.c_int32), ("have_prev_D", ctypes.c_int32),
                ("prev_D_size", ctypes.c_int64)]


class trd_profile(ctypes.Structure):
    _fields_ = [("pass1_ms", ctypes.c_double), ("pass2_ms", ctypes.c_double),
                ("pass1_launches", ctypes.c_int64), ("pass2_launches", ctypes.c_int64),
                ("pass1_entries", ctypes.c_double), ("pass2_entries", ctypes.c_double),
                ("pass1_flops", ctypes.c_double), ("pass2_flops", ctypes.c_double),
                ("pass1_bytes", ctypes.c_double), ("pass2_bytes", ctypes.c_double),
                ("pass1_mma_flops", ctypes.c_double), ("pass2_mma_flops", ctypes.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libtrd.so (built in-tree by paper_2305_09044_b200/build.py).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libtrd.so not built at {path}; run python -m paper_2305_09044_b200.build")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    P, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "trd_init": (i32, [ctypes.POINTER(trd_config), ctypes.POINTER(trd_shard), P, P, P]),
        "trd_init_ex": (i32, [ctypes.POINTER(trd_config), ctypes.POINTER(trd_shard), P, P,
                              ctypes.POINTER(trd_exchange), P]),
        "trd_upload": (i32, [P, P, P]),
        "trd_sketch": (i32, [P, i32, i32, P, P]),
        "trd_sweep": (i32, [P, i32, P]),
        "trd_reconstruct": (i32, [P, P, i64, P]),
        "trd_error": (i32, [P, P, P, d, ctypes.POINTER(trd_error_stats)]),
        "trd_get_cores": (i32, [P, P]),
        "trd_set_cores": (i32, [P, P]),
        "trd_get_state": (i32, [P, ctypes.POINTER(trd_state), P]),
        "trd_set_state": (i32, [P, ctypes.POINTER(trd_state), P]),
        "trd_block_probe": (i32, [P, i32, i32, P, P, P, P]),
        "trd_launch_count": (i64, [P]),
        "trd_set_profiling": (i32, [P, i32]),
        "trd_get_profile": (i32, [P, ctypes.POINTER(trd_profile)]),
        "trd_nccl_unique_id": (i32, [P]),
        "trd_destroy": (None, [P]),
        "trd_last_error": (ctypes.c_char_p, [P]),
        "trd_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        if path != os.path.join(HERE, "libtrd.so") and not hasattr(lib, name):
            continue        # A/B experiments (TRD_LIB_PATH): an older library may lack newer calls
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def declared_symbols(header: str = HEADER) -> List[str]:
    """Names of the entry points include/trd.h declares (TRD_API functions)."""
    import re
    txt = open(header).read()
    return sorted(set(re.findall(r"TRD_API\s+[\w\s\*]+?\b(trd_\w+)\s*\(", txt)))


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.trd_nccl_unique_id(buf)
    if st != 0:
        raise TrdError(st, "trd_nccl_unique_id")
    return buf.raw


def _ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class TRD:
    """One libtrd context (trd_init ... trd_destroy).

    values / mask: torch tensors (device, or pinned host when host=True) holding the local
    shard: values float32 (dense or packed), mask int32/uint32 bit words.
    init_cores: list of float32 arrays (r_k, I_k, r_{k+1}).
    """

    def __init__(self, dims, ranks, values, mask, init_cores, *, sigma_mode=TRD_SIGMA_RMS,
                 sigma=1.0, sigma_theta=1.0, sigma_min=1e-3, lambda_rel=1e-6, step=0.0,
                 sketch=None, seed=0, shard_mode=0, shard_range=None, world=1, rank=0,
                 nccl_id: Optional[bytes] = None, packed=False, host=False, stream=None,
                 scaling=0, sampling=0, exchange=None):
        import torch
        self.lib = load_library()
        N = len(dims)
        cfg = trd_config()
        cfg.order = N
        for m in range(N):
            cfg.dims[m] = int(dims[m])
            cfg.ranks[m] = int(ranks[m])
            cfg.sketch[m] = int(sketch[m]) if sketch is not None else 0
        cfg.sigma_mode = int(sigma_mode)
        cfg.sigma = float(sigma)
        cfg.sigma_theta = float(sigma_theta)
        cfg.sigma_min = float(sigma_min)
        cfg.lambda_rel = float(lambda_rel)
        cfg.step = float(step)
        cfg.seed = int(seed) & ((1 << 64) - 1)
        cfg.shard_mode = int(shard_mode)
        cfg.world = int(world)
        cfg.rank = int(rank)
        cfg.scaling = int(scaling)
        cfg.sampling = int(sampling)
        self._nccl_buf = None
        if nccl_id is not None:
            self._nccl_buf = ctypes.create_string_buffer(nccl_id, 128)
            cfg.nccl_unique_id = ctypes.cast(self._nccl_buf, ctypes.c_void_p)
        sh = trd_shard()
        if shard_range is None:
            shard_range = (0, int(dims[shard_mode]))
        sh.shard_begin, sh.shard_end = int(shard_range[0]), int(shard_range[1])
        sh.values = _ptr(values)
        sh.mask_bits = _ptr(mask)
        sh.packed = 1 if packed else 0
        sh.host = 1 if host else 0
        self._keep = (values, mask)
        self.N = N
        self.dims = [int(x) for x in dims]
        self.sampling = int(sampling)
        self.sketch_sizes = [int(sketch[m]) if sketch is not None else 0 for m in range(N)]
        self.ranks = [int(x) for x in ranks]
        cores = [np.ascontiguousarray(c, dtype=np.float32) for c in init_cores]
        arr = (ctypes.c_void_p * N)(*[c.ctypes.data for c in cores])
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        self.stream = stream
        self.ctx = ctypes.c_void_p()
        if exchange is not None:
            # exchange(buf_dev_ptr, n, op, stream) -> None: an in-place allreduce of n doubles
            def _cb(user, buf, n, op, strm):
                try:
                    exchange(int(buf or 0), int(n), int(op), int(strm or 0))
                    return 0
                except Exception:                                  # reported as TRD_ERR_NCCL
                    import traceback
                    traceback.print_exc()
                    return 1
            self._ex_cb = ALLREDUCE_FN(_cb)
            self._ex = trd_exchange(self._ex_cb, None)
            st = self.lib.trd_init_ex(ctypes.byref(cfg), ctypes.byref(sh), arr, ctypes.c_void_p(stream),
                                      ctypes.byref(self._ex), ctypes.byref(self.ctx))
        else:
            st = self.lib.trd_init(ctypes.byref(cfg), ctypes.byref(sh), arr, ctypes.c_void_p(stream),
                                   ctypes.byref(self.ctx))
        if st != 0:
            raise TrdError(st, "trd_init")

    # ------------------------------------------------------------------
    def _check(self, st, what):
        if st != 0:
            raise TrdError(st, f"{what}: {self.lib.trd_last_error(self.ctx).decode()}")

    def sweep(self, n: int = 1, stats: bool = True):
        if not stats:
            self._check(self.lib.trd_sweep(self.ctx, int(n), None), "trd_sweep")
            return None
        recs = (trd_sweep_stats * n)()
        self._check(self.lib.trd_sweep(self.ctx, int(n), recs), "trd_sweep")
        out = []
        for r in recs:
            out.append(dict(sigma=r.sigma, sum_e2=r.sum_e2, welsch=r.welsch_loss, stop_e=r.stop_e,
                            ms=r.ms, n_obs=r.n_obs, eta=list(r.eta)[:self.N], num=list(r.num)[:self.N],
                            den=list(r.den)[:self.N], nnz=list(r.nnz)[:self.N],
                            skipped=r.skipped_mask, replica_mismatch=r.replica_mismatch))
        return out

    def sketch(self, t: int, k: int):
        import torch
        total = sum(self.dims)
        if self.sampling == TRD_SAMPLING_ROWS:         # J draws in every mode but k
            J = 1
            for m in range(self.N):
                if m != k:
                    s_m = self.sketch_sizes[m]
                    J *= self.dims[m] if (s_m <= 0 or s_m >= self.dims[m]) else s_m
            total = self.dims[k] + (self.N - 1) * J
        buf = torch.empty(total, dtype=torch.int32, device="cuda")
        sizes = (ctypes.c_int64 * TRD_MAX_ORDER)()
        self._check(self.lib.trd_sketch(self.ctx, int(t), int(k), ctypes.c_void_p(buf.data_ptr()),
                                        sizes), "trd_sketch")
        host = buf.cpu().numpy()
        out, off = [], 0
        for m in range(self.N):
            out.append(host[off:off + sizes[m]].astype(np.int64))
            off += sizes[m]
        return out

    def reconstruct(self, lin_idx):
        import torch
        out = torch.empty(lin_idx.numel(), dtype=torch.float32, device=lin_idx.device)
        self._check(self.lib.trd_reconstruct(self.ctx, ctypes.c_void_p(lin_idx.data_ptr()),
                                             int(lin_idx.numel()), ctypes.c_void_p(out.data_ptr())),
                    "trd_reconstruct")
        return out

    def error(self, ref, eval_bits=None, peak=1.0):
        es = trd_error_stats()
        self._check(self.lib.trd_error(self.ctx, ctypes.c_void_p(_ptr(ref)),
                                       ctypes.c_void_p(_ptr(eval_bits)), float(peak), ctypes.byref(es)),
                    "trd_error")
        return dict(rel_err_all=es.rel_err_all, rel_err_observed=es.rel_err_observed,
                    psnr=es.psnr, n_eval=es.n_eval)

    def get_cores(self):
        N = self.N
        cores = [np.empty((self.ranks[k], self.dims[k], self.ranks[(k + 1) % N]), dtype=np.float32)
                 for k in range(N)]
        arr = (ctypes.c_void_p * N)(*[c.ctypes.data for c in cores])
        self._check(self.lib.trd_get_cores(self.ctx, arr), "trd_get_cores")
        return cores

    def set_cores(self, cores):
        cores = [np.ascontiguousarray(c, dtype=np.float32) for c in cores]
        arr = (ctypes.c_void_p * self.N)(*[c.ctypes.data for c in cores])
        self._check(self.lib.trd_set_cores(self.ctx, arr), "trd_set_cores")

    def get_state(self):
        """Iteration state beyond the cores (sigma, sweep counter t, D^{t-1}) for an exact resume."""
        In = self.dims[self.N - 1]
        prev = np.zeros((In, In))
        st = trd_state()
        self._check(self.lib.trd_get_state(self.ctx, ctypes.byref(st), prev.ctypes.data), "trd_get_state")
        return dict(sigma=st.sigma, sweep=st.sweep, have_prev_D=st.have_prev_D,
                    prev_D=prev if st.have_prev_D else None)

    def set_state(self, state):
        In = self.dims[self.N - 1]
        prev = state.get("prev_D")
        st = trd_state(float(state["sigma"]), int(state["sweep"]), int(state["have_prev_D"]), In * In)
        buf = None if prev is None else np.ascontiguousarray(prev, dtype=np.float64)
        self._check(self.lib.trd_set_state(self.ctx, ctypes.byref(st), None if buf is None else buf.ctypes.data),
                    "trd_set_state")

    def upload(self, values_host, mask_host):
        self._check(self.lib.trd_upload(self.ctx, ctypes.c_void_p(_ptr(values_host)),
                                        ctypes.c_void_p(_ptr(mask_host))), "trd_upload")

    def block_probe(self, t: int, k: int):
        Ik = self.dims[k]
        R2 = self.ranks[k] * self.ranks[(k + 1) % self.N]
        d = np.zeros((Ik, R2))
        G = np.zeros((R2, R2))
        h = np.zeros((Ik, R2))
        st5 = np.zeros(5)
        self._check(self.lib.trd_block_probe(self.ctx, int(t), int(k), d.ctypes.data, G.ctypes.data,
                                             h.ctypes.data, st5.ctypes.data), "trd_block_probe")
        return dict(d=d, G=G, h=h, sum_e2=st5[0], n_obs=st5[1], welsch=st5[2], num=st5[3], den=st5[4])

    def set_profiling(self, on: bool):
        self._check(self.lib.trd_set_profiling(self.ctx, 1 if on else 0), "trd_set_profiling")

    def get_profile(self):
        p = trd_profile()
        self._check(self.lib.trd_get_profile(self.ctx, ctypes.byref(p)), "trd_get_profile")
        return {f: getattr(p, f) for f, _ in trd_profile._fields_}

    @property
    def launch_count(self) -> int:
        return int(self.lib.trd_launch_count(self.ctx))

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            self.lib.trd_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
