"""In-tree build of libcoolchic_b200.so (sm_100a) and the oracle checkers.

nvcc compiles every csrc/*.cu for ``-gencode arch=compute_100a,code=sm_100a``
with -lineinfo (ncu source view) and WITHOUT --use_fast_math (parity needs IEEE
division/sqrt and the reference's polynomial transcendentals).  Objects are
rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
OUT = PKG / "libcoolchic_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", str(REPO / "include")]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_product(verbose: bool = False, ptxas_v: bool = False) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((REPO / "include").glob("*.h"))
    objs, cmds = [], []
    for src in sorted(CSRC.glob("*.cu")):
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if _newer(obj, [src, *headers]) or ptxas_v:
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
            if ptxas_v:
                cmd.insert(1, "-Xptxas=-v")
            cmds.append(cmd)
    if cmds:
        from concurrent.futures import ThreadPoolExecutor

        def run(cmd):
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)

        with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
            list(ex.map(run, cmds))
    if _newer(OUT, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(OUT), *map(str, objs), "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return OUT


def build_oracle(verbose: bool = False) -> None:
    """The checkers: the plain-C port always; the reference build only where
    /root/reference exists (it never exists on the GPU box, whose copy of
    oracle/_ref/*.so was built here and travels with the snapshot)."""
    make = shutil.which("make")
    odir = REPO / "oracle"
    if make is None:
        raise RuntimeError("make not found")
    targets = ["port"]
    if Path("/root/reference/proj/include/coolcodec/encoder.hpp").exists():
        targets += ["ref", "dropin"]
    subprocess.run([make, "-s", "-C", str(odir), *targets], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    verbose = "-v" in argv
    build_product(verbose=verbose, ptxas_v="--ptxas" in argv)
    if "--no-oracle" not in argv:
        build_oracle(verbose=verbose)


if __name__ == "__main__":
    main()
