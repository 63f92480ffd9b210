"""Build libnwb200.so (sm_100a) in-tree with nvcc.

Every translation unit is compiled for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` (ncu source view) and linked into one shared library next
to this file, so it travels to the GPU box with the repo snapshot.
``tables.cu`` is compiled with ``-fmad=false``: the multiplier tables must
round like numpy (no contraction into FMAs).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB_NAME = "libnwb200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)
BUILD_DIR = os.path.join(os.path.dirname(HERE), "build", "nwb200")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
          "--expt-relaxed-constexpr", "-I", CSRC, "-I", INCLUDE]
# (object, source, extra flags): spectral.cu is split by part and type so its
# FFT instantiations compile in parallel
UNITS = [
    ("spectral_theta_f64", "spectral.cu", ["-DNWB_SPEC_PART=1", "-DNWB_SPEC_T=double"]),
    ("spectral_theta_f32", "spectral.cu", ["-DNWB_SPEC_PART=1", "-DNWB_SPEC_T=float"]),
    ("spectral_rho_f64", "spectral.cu", ["-DNWB_SPEC_PART=2", "-DNWB_SPEC_T=double"]),
    ("spectral_rho_f32", "spectral.cu", ["-DNWB_SPEC_PART=2", "-DNWB_SPEC_T=float"]),
    ("weno", "weno.cu", []),
    ("capi", "capi.cu", []),
    ("tables", "tables.cu", ["-fmad=false"]),
    ("splitting", "splitting.cu", ["-fmad=false"]),
    ("metrics", "metrics.cu", []),
]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: the B200 library cannot be built")
    return path


def _sources():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(INCLUDE, "nwb200.h"))
    return deps


STAMP = LIB_PATH + ".defines"


def up_to_date() -> bool:
    if not os.path.exists(LIB_PATH):
        return False
    # a library built with experiment defines is never the default build
    if os.path.exists(STAMP) and open(STAMP).read().strip():
        return False
    t = os.path.getmtime(LIB_PATH)
    return all(os.path.getmtime(d) <= t for d in _sources())


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
          defines=(), out: str | None = None) -> str:
    """Compile and link; ``defines`` build an experiment variant, which must be
    written elsewhere (``out``) so the default library is never a variant."""
    if defines and out is None:
        raise ValueError("experiment defines need an explicit out= library path")
    lib_path = out or LIB_PATH
    if not force and not defines and out is None and up_to_date():
        return LIB_PATH
    # variants get their own object directory, keyed by the whole output path
    tag = os.path.abspath(lib_path).replace(".so", "").strip(os.sep).replace(os.sep, "_")
    build_dir = BUILD_DIR + ("_" + tag if out else "")
    os.makedirs(build_dir, exist_ok=True)
    os.makedirs(os.path.dirname(os.path.abspath(lib_path)), exist_ok=True)
    objs = []
    procs = []
    headers = [d for d in _sources() if not d.endswith(".cu")]
    newest_header = max(os.path.getmtime(h) for h in headers)
    for name, unit, extra in UNITS:
        obj = os.path.join(build_dir, name + ".o")
        objs.append(obj)
        src = os.path.join(CSRC, unit)
        # incremental: an object is reused when newer than its source and every header
        # (experiment variants and forced builds recompile everything)
        if (not force and not defines and out is None and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), newest_header)):
            continue
        cmd = [nvcc(), *ARCH, *COMMON, *extra, *[f"-D{d}" for d in defines], "-c",
               os.path.join(CSRC, unit), "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((name, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                             text=True)))
    failed = []
    for unit, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose or ptxas_v:
            print(out, file=sys.stderr)
        if p.returncode != 0:
            failed.append(unit)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = lib_path + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib_path)
    with open(lib_path + ".defines", "w") as fh:
        fh.write(" ".join(defines))
    return lib_path


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                ptxas_v="--ptxas" in sys.argv, defines=defs, out=outs[0] if outs else None))
