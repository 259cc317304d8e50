"""Build libquadb200.so (sm_100a) in-tree with nvcc.

    python -m paper_2407_14783_b200.build [--force] [-v]

Each csrc/*.cu is compiled to an object for ``-gencode
arch=compute_100a,code=sm_100a`` with -lineinfo (so ncu's source page maps to
the code) and linked into paper_2407_14783_b200/libquadb200.so with the CUDA
runtime linked statically; the .so travels to the GPU box with the repo.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libquadb200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "-Xptxas", "-warn-spills", f"-I{INCLUDE}", f"-I{CSRC}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _host_compiler_flags():
    # the image's default CC wrapper lacks some specs; point nvcc at the system g++
    for cxx in ("/usr/bin/g++-13", "/usr/bin/g++"):
        if os.path.exists(cxx):
            return ["-ccbin", cxx]
    return []


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def needs_build() -> bool:
    return not os.path.exists(LIB) or os.path.getmtime(LIB) < _deps_mtime()


def build(force: bool = False, verbose: bool = False, extra_flags=()) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    cc = nvcc()
    hostc = _host_compiler_flags()

    # a translation unit is recompiled when it, a header or this script is newer
    # than its object (or always, with extra flags: tuning builds)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")]
    headers += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)] + [os.path.abspath(__file__)]
    common = max(os.path.getmtime(f) for f in headers)
    stamp = os.path.join(OBJ, "flags.txt")  # objects of a tuning build (-D ...) are never reused by another build
    flags_now = " ".join(extra_flags)
    if not os.path.exists(stamp) or open(stamp).read() != flags_now:
        force = True

    def compile_one(src):
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(common, os.path.getmtime(os.path.join(CSRC, src)))):
            return obj
        cmd = [cc, *ARCH, *NVCC_FLAGS, *hostc, *extra_flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, flush=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    with open(stamp, "w") as f:
        f.write(flags_now)
    tmp = LIB + ".tmp"
    cmd = [cc, *ARCH, *hostc, "-shared", "-cudart", "static", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true", help="print register/spill usage")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra preprocessor define (tuning)")
    a = ap.parse_args(argv)
    extra = (["-Xptxas", "-v"] if a.ptxas_v else []) + [f"-D{d}" for d in a.defines]
    print(build(force=a.force or a.ptxas_v or bool(a.defines), verbose=a.verbose or a.ptxas_v, extra_flags=extra))


if __name__ == "__main__":
    sys.exit(main())
