"""Build libb2mhd.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libb2mhd.so")
# Experimental variants (e.g. B2_ZM_TX64=16) build to libb2mhd_<tag>.so; load with B2MHD_LIB=<path>.
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import site
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        inc = os.path.join(sp, "nvidia", "nccl", "include")
        lib = os.path.join(sp, "nvidia", "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("NCCL headers/library (nvidia-nccl wheel) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(INCLUDE, "b2mhd.h"), os.path.abspath(__file__)]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, defines=None, lib=None) -> str:
    global LIB
    if lib:
        LIB = lib
    if not force and up_to_date():
        return LIB
    inc, lib = nccl_dirs()
    objdir = os.path.join(HERE, "build" + ("_" + "_".join(defines) if defines else ""))
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-I", inc, "-I", INCLUDE,
              "--expt-relaxed-constexpr"] + ARCH + ["-D" + d for d in (defines or [])]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, "-c", src, "-o", obj] + common
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), cmd))
        objs.append(obj)
    for p, cmd in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out.decode())
        if p.returncode:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, "-shared", "-o", LIB + ".tmp"] + objs + ARCH + \
        ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    subprocess.check_call(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    tag = "_".join(d.replace("=", "") for d in defs)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs or None,
                lib=os.path.join(HERE, f"libb2mhd_{tag}.so") if defs else None))
