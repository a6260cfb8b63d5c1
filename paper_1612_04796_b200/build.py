"""Build the in-tree C-ABI shared library libpmgdg.so for sm_100a (nvcc, no JIT cache)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpmgdg.so")
SOURCES = ["api.cu", "kern_fdm.cu", "kern_fdm_ct.cu", "kern_fdm_dl.cu", "kern_apply.cu", "kern_apply33.cu", "kern_xfer.cu", "kern_global.cu", "kern_misc.cu",
           "setup.cpp", "probe.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "pmg_dg.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, extra=(), out=None):
    """extra / out: diagnostic variants (-D switches) built into their own object dir and .so."""
    lib = out or LIB
    objdir = os.path.join(HERE, "build", os.path.basename(lib) + ".obj") if out else os.path.join(HERE, "build")
    if not out and not force and not _stale():
        return LIB
    os.makedirs(objdir, exist_ok=True)

    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    headers.append(os.path.join(ROOT, "include", "pmg_dg.h"))

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        if not force and os.path.exists(obj):
            t = os.path.getmtime(obj)
            if all(os.path.getmtime(d) <= t for d in headers + [os.path.join(CSRC, src)]):
                return obj, subprocess.CompletedProcess([], 0, "", "")
        cmd = [NVCC] + FLAGS + list(extra) + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-x", "cu"] + FLAGS + list(extra) + ["-c", os.path.join(CSRC, src), "-o", obj]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    # translation units compile in parallel (the kernel files dominate the build time)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = []
    for src, (obj, r) in zip(SOURCES, results):
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed on " + src)
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    r = subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs
                       + ["-lcudart"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH -DFOO=1 ...]   (variants: always a full rebuild)
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    extra = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args or out is not None, verbose="-v" in args, extra=extra, out=out))
