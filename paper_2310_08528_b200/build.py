"""Build libfgs.so (all CUDA sources of csrc/) in-tree for sm_100a with nvcc.

`python -m paper_2310_08528_b200.build` or `__graft_entry__.build()`.  Explicit
-gencode arch=compute_100a,code=sm_100a (plain -arch=sm_100a emits compute_100
PTX on which ptxas rejects tcgen05.*).
"""
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfgs.so")
# checked variant: the same sources with -DFGS_CHECKED (device-side bounds / invariant assertions and an
# mbarrier watchdog, csrc/fgs_internal.cuh); loaded instead of libfgs.so when FGS_LIB=checked
LIB_CHECKED = os.path.join(HERE, "libfgs_checked.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "-Xptxas", "-v"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "fgs.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, checked=None):
    """Compile libfgs.so (checked=True: libfgs_checked.so; None: the one FGS_LIB selects) if it is
    missing or older than its sources.  Safe to call from several processes at once (torchrun ranks):
    one builds under an exclusive file lock, the others wait and then find the library up to date."""
    if checked is None:
        checked = os.environ.get("FGS_LIB", "") == "checked"
    lib = LIB_CHECKED if checked else LIB
    if not force and not needs_build(lib):
        return lib
    import fcntl
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    with open(os.path.join(HERE, "build", ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and not needs_build(lib):
                return lib
            return _build(verbose, checked, force)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build(verbose=False, checked=False, force=False):
    nvcc = nvcc_path()
    objdir = os.path.join(HERE, "build", "checked") if checked else os.path.join(HERE, "build")
    LIB_OUT = LIB_CHECKED if checked else LIB
    os.makedirs(objdir, exist_ok=True)
    objs = []
    logs = []
    procs = []
    # incremental: an object newer than its source, every header and this file is reused (its ptxas log
    # is kept beside it); experiment builds (FGS_NVCC_EXTRA) and force=True always recompile
    extra = os.environ.get("FGS_NVCC_EXTRA", "").split()
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "fgs.h"), __file__]
    stamp = os.path.join(objdir, ".plain")      # present when the objects came from a build without extras
    reuse_ok = not force and not extra and os.path.exists(stamp)
    if os.path.exists(stamp):
        os.remove(stamp)
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if reuse_ok and os.path.exists(obj) and os.path.exists(obj + ".log") and all(
                os.path.getmtime(d) < os.path.getmtime(obj) for d in [src] + hdrs):
            procs.append((src, obj, None))
            continue
        # FGS_NVCC_EXTRA: extra flags for experiments (e.g. -D switches); not set in normal builds
        cmd = ([nvcc] + NVCC_FLAGS + (["-DFGS_CHECKED"] if checked else []) + extra + ["-c", src, "-o", obj])
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, obj, p in procs:
        if p is None:
            with open(obj + ".log") as fh:
                logs.append(fh.read())
            objs.append(obj)
            continue
        out = p.communicate()[0].decode(errors="replace")
        logs.append(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        with open(obj + ".log", "w") as fh:
            fh.write(out)
        objs.append(obj)
    if not extra:
        open(stamp, "w").close()
    tmp = LIB_OUT + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", tmp] + objs + ["-cudart", "static"]
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if p.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + p.stdout.decode(errors="replace"))
    os.replace(tmp, LIB_OUT)
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
