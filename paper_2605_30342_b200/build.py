"""Build the native library in-tree: nvcc, sm_100a only.

    python -m paper_2605_30342_b200.build          # -> paper_2605_30342_b200/libgavis_b200.so

Every translation unit is compiled with -fmad=false: the fp64 expressions that
feed the reference's discrete decisions must round exactly like its
(unfused, -O3, no -march) double code. Kernels request FMA explicitly where it
is wanted (__fmaf_rn in the fp32 colour dot product).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "native")
LIB = os.path.join(PKG, "libgavis_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-O3",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False, defines=(), lib: str = LIB,
          build_dir: str = BUILD) -> str:
    """Compile every csrc/*.cu and link `lib`. `defines` (e.g. ["GAVIS_EXACT_BATCH=96"])
    with a separate `lib`/`build_dir` build an A/B variant of the compile-time knobs
    (loaded through GAVIS_LIB_PATH)."""
    os.makedirs(build_dir, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    objs = []
    jobs = []
    for src in sources:
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if _stale(obj, [src] + headers + [__file__]):
            cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0 or verbose or ptxas_info:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cmd[-3]}")

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(lib):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib


if __name__ == "__main__":
    # python -m paper_2605_30342_b200.build [-v] [--ptxas] [--variant NAME -DKNOB=V ...]
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        print(build(verbose="-v" in args, ptxas_info="--ptxas" in args, defines=defs,
                    lib=os.path.join(ROOT, "build", f"libgavis_b200_{name}.so"),
                    build_dir=os.path.join(ROOT, "build", f"native_{name}")))
    else:
        print(build(verbose="-v" in args, ptxas_info="--ptxas" in args, defines=defs))
