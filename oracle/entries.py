"""Entry-wise data source of the float64 oracle (full-size problems).

TEST INFRASTRUCTURE ONLY (see trd_oracle.py): only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.

The dense oracle path (trd_oracle.DenseSource) unfolds the sketch X_I into an I_k x J matrix,
which does not fit for the 80^5 configs.  This source instead visits the observed entries of
the sketch one by one in C (oracle/trd_entries.c, plain float64 loops over Thm 1's subchain
S(j) and Eq. 7 / 9 / 12 per entry), with OpenMP over the first subchain mode.  The two
forms compute the same sums (pinned: tests/test_oracle_pins.py, dense vs entry-wise on
random problems, <= 1e-12).
"""
import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "trd_entries.c")
LIB = os.path.join(HERE, "_build", "libtrd_entries.so")
# plain float64: no fast-math, no FMA contraction
CFLAGS = ["-O3", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math"]

_lib = None
_lock = threading.Lock()


def build(force=False):
    """Compile trd_entries.c into oracle/_build/ (gcc; test infrastructure, not the product)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + ".%d.tmp" % os.getpid()
    subprocess.run(["gcc"] + CFLAGS + [SRC, "-o", tmp, "-lm"], check=True)
    os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            P = ctypes.c_void_p
            L.oc_block_pass.restype = ctypes.c_int
            L.oc_block_pass.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, P,
                                        P, ctypes.c_double, ctypes.c_int, P, P, P, P, ctypes.c_int64]
            L.oc_reconstruct.restype = ctypes.c_int
            L.oc_reconstruct.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_int64, P]
            _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Cores:
    """Keeps float64 C-contiguous copies of the cores and an array of their pointers."""

    def __init__(self, cores):
        self.arrs = [np.ascontiguousarray(c, dtype=np.float64) for c in cores]
        self.ptrs = (ctypes.c_void_p * len(self.arrs))(*[a.ctypes.data for a in self.arrs])


class EntrySource:
    """Observed entries of X (mask bits over the global linear order, Def. 2),
    values dense (values[lin]) or packed (n-th observed entry at values[n])."""

    def __init__(self, dims, mask_words, values, packed):
        self.dims = [int(d) for d in dims]
        self.mask = np.ascontiguousarray(np.asarray(mask_words).view(np.uint32))
        self.values = np.ascontiguousarray(np.asarray(values, dtype=np.float32))
        self.packed = bool(packed)
        if self.packed:
            cnt = np.bitwise_count(self.mask).astype(np.uint64)
            self.prefix = np.concatenate([[np.uint64(0)], np.cumsum(cnt[:-1], dtype=np.uint64)])
        else:
            self.prefix = None
        self.n_obs = int(np.bitwise_count(self.mask).sum())
        self._dims = np.asarray(self.dims, dtype=np.int64)

    # -- the two per-entry sums of block k (Eq. 7 + Eq. 9/15; Eq. 12/18) ------------------
    def _call(self, pass_, cores, k, sets, ranks, sigma, sigma_inf, h=None, want_abs=False):
        N = len(self.dims)
        C = _Cores(cores)
        rk = np.asarray(ranks, dtype=np.int32)
        sets64 = [np.ascontiguousarray(s, dtype=np.int64) for s in sets]
        sptr = (ctypes.c_void_p * N)(*[s.ctypes.data for s in sets64])
        sizes = np.asarray([len(s) for s in sets64], dtype=np.int64)
        R2 = int(ranks[k]) * int(ranks[(k + 1) % N])
        d = np.zeros((self.dims[k], R2), dtype=np.float64)
        st = np.zeros(4, dtype=np.float64)
        cap = 0
        abs_e = None
        if want_abs:
            cap = 1
            for s in sets64:
                cap *= len(s)
            cap = min(cap, self.n_obs)
            abs_e = np.zeros(max(cap, 1), dtype=np.float64)
        hh = None if h is None else np.ascontiguousarray(h, dtype=np.float64)
        r = lib().oc_block_pass(pass_, N, k, _ptr(self._dims), _ptr(rk), C.ptrs, sptr, _ptr(sizes),
                                _ptr(self.mask), _ptr(self.values),
                                _ptr(self.prefix) if self.packed else None,
                                float(sigma), 1 if sigma_inf else 0,
                                None if hh is None else _ptr(hh), _ptr(d), _ptr(st),
                                None if abs_e is None else _ptr(abs_e), ctypes.c_int64(cap))
        if r != 0:
            raise RuntimeError("oc_block_pass failed")
        return d, st, abs_e

    def pass1(self, cores, k, sets, ranks, sigma, sigma_inf, want_abs=False):
        """d (I_k x R_k^2, column c + r_k b), sum_e2, welsch, n, |e| of the observed entries."""
        d, st, abs_e = self._call(1, cores, k, sets, ranks, sigma, sigma_inf, want_abs=want_abs)
        n = int(round(st[2]))
        return d, float(st[0]), float(st[1]), n, (abs_e[:n] if want_abs else None)

    def pass2(self, cores, k, sets, ranks, sigma, sigma_inf, h):
        """den = sum over the observed sketch entries of w (h(i_k) . S(j))^2 (Eq. 12/18)."""
        _, st, _ = self._call(2, cores, k, sets, ranks, sigma, sigma_inf, h=h)
        return float(st[3])

    def reconstruct(self, cores, ranks, lin):
        """Def. 1 at the given global linear indices."""
        C = _Cores(cores)
        lin = np.ascontiguousarray(lin, dtype=np.int64)
        out = np.zeros(len(lin), dtype=np.float64)
        r = lib().oc_reconstruct(len(self.dims), _ptr(self._dims), _ptr(np.asarray(ranks, dtype=np.int32)),
                                 C.ptrs, _ptr(lin), ctypes.c_int64(len(lin)), _ptr(out))
        if r != 0:
            raise RuntimeError("oc_reconstruct failed")
        return out
