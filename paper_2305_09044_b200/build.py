"""Build libtrd.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtrd.so")
# checked build (-DTRD_CHECKED=1): device invariant checks, mbarrier watchdog, schedule fuzzing
# (tests/test_gpu_checked.py loads it in a subprocess via TRD_LIB_PATH)
CHECKED_LIB = os.path.join(HERE, "libtrd_checked.so")
SOURCES = ["trd_kernels.cu", "trd_tc.cu", "trd_big.cu", "trd_api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
           [os.path.join(HERE, "..", "include", "trd.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """Compile the sources (in parallel) and link libtrd.so.  `out` / `defines` (-D flags) are
    for kernel-variant experiments only; the product library is LIB with the default macros."""
    lib = out or LIB
    if out is None and not defines and not force and not needs_build():
        return LIB
    tag = "" if out is None else "_" + os.path.basename(out).replace(".so", "")
    procs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", tag + ".o"))
        cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + objs + ["-ldl"]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return lib


def build_all(force=False):
    """The product library and the checked library, built concurrently."""
    import threading
    errs = []

    def run(kw):
        try:
            build(**kw)
        except Exception as e:   # re-raised below
            errs.append(e)

    need_checked = force or not os.path.exists(CHECKED_LIB) or \
        os.path.getmtime(CHECKED_LIB) < max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC))
    ts = [threading.Thread(target=run, args=(dict(force=force),))]
    if need_checked:
        ts.append(threading.Thread(target=run, args=(dict(out=CHECKED_LIB, defines=("TRD_CHECKED=1",)),)))
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return LIB, CHECKED_LIB


if __name__ == "__main__":
    # python -m paper_2305_09044_b200.build [--force] [--out PATH -DNAME=V ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    build(force="--force" in args, verbose=True, out=out, defines=defs)
