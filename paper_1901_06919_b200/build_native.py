"""Build libfdl_b200.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libfdl_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(CSRC.glob("*.cu"))


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = True) -> Path:
    if not force and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for src in sources():
        obj = OUT.parent / (src.stem + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-O3", "-I", str(ROOT / "include"), "-I", str(CSRC),
               *os.environ.get("FDL_NVCC_EXTRA", "").split(),  # A/B experiments (-D...)
               "-c", str(src), "-o", str(obj)]
        jobs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(str(obj))
    failed = False
    for src, proc in jobs:
        out, _ = proc.communicate()
        if proc.returncode != 0:
            failed = True
            sys.stderr.write(out.decode())
            sys.stderr.write(f"nvcc failed on {src.name}\n")
        elif verbose and out.strip():
            sys.stderr.write(out.decode())
    if failed:
        raise RuntimeError("nvcc compilation failed")
    link = [NVCC, *ARCH, "-shared", "-o", str(OUT), *objs, "-lcufft",
            "-L/usr/local/cuda/lib64", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(link, check=True)
    for o in objs:
        os.remove(o)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(OUT)
