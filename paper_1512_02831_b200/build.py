"""Build libbkt.so (the sm_100a engine) in-tree.

    python -m paper_1512_02831_b200.build [--jobs N] [--force]

Compiles every translation unit of csrc/ with nvcc for sm_100a
(-gencode arch=compute_100a,code=sm_100a -lineinfo), one leafscan object per
kernel dimensionality (dims.h BKT_DIM_LIST) in parallel, and links them into
paper_1512_02831_b200/_lib/libbkt.so.  Objects are cached under
paper_1512_02831_b200/_lib/obj/ and rebuilt when a source or header changes.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
OBJ_DIR = LIB_DIR / "obj"
LIB = LIB_DIR / "libbkt.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", str(CSRC),
                  "-I", str(INCLUDE), "--expt-relaxed-constexpr"]


def _dims() -> list[int]:
    text = (CSRC / "dims.h").read_text()
    body = text.split("#define BKT_DIM_LIST(X)")[1].split("\n\n")[0]
    return [int(x) for x in re.findall(r"X\((\d+)\)", body)]


def _sources_hash(extra: str) -> str:
    h = hashlib.sha256(extra.encode())
    for p in sorted(list(CSRC.glob("*")) + [INCLUDE / "bkt.h"]):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(NVFLAGS).encode())
    return h.hexdigest()[:16]


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    tag = _sources_hash("v1")
    stamp = LIB_DIR / "libbkt.stamp"
    if LIB.exists() and stamp.exists() and stamp.read_text() == tag and not force:
        return LIB
    units: list[tuple[list[str], Path]] = []
    for d in _dims():
        obj = OBJ_DIR / f"leafscan_d{d}.o"
        units.append(([NVCC, *NVFLAGS, f"-DBKT_D={d}", "-c", str(CSRC / "leafscan_inst.cu"), "-o", str(obj)], obj))
    for src in ("engine.cu", "misc.cu", "leafscan_tc_inst.cu"):
        obj = OBJ_DIR / (Path(src).stem + ".o")
        units.append(([NVCC, *NVFLAGS, "-c", str(CSRC / src), "-o", str(obj)], obj))
    obj = OBJ_DIR / "build_tree.o"
    units.append((["g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-I", str(INCLUDE), "-c",
                   str(CSRC / "build_tree.cpp"), "-o", str(obj)], obj))
    jobs = jobs or max(1, os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        list(ex.map(lambda u: _run(u[0]), units))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "--cudart", "static", "-o", str(tmp), *[str(u[1]) for u in units], "-lpthread"])
    os.replace(tmp, LIB)
    stamp.write_text(tag)
    if verbose:
        print(f"built {LIB}")
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(a.jobs, a.force, verbose=True)


if __name__ == "__main__":
    sys.exit(main())
