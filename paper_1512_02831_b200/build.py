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


def _deps(src: Path, seen: set | None = None) -> set:
    """src plus every local header it includes (transitively)."""
    seen = set() if seen is None else seen
    if src in seen or not src.exists():
        return seen
    seen.add(src)
    for inc in re.findall(r'#include\s+"([^"]+)"', src.read_text()):
        for base in (src.parent, CSRC, INCLUDE):
            cand = (base / inc).resolve()
            if cand.exists():
                _deps(cand, seen)
                break
    return seen


def _unit_hash(cmd: list[str], src: Path) -> str:
    h = hashlib.sha256(" ".join(cmd).encode())
    for p in sorted(_deps(src)):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def _compile(cmd: list[str], src: Path, obj: Path, force: bool) -> bool:
    """Compile one unit unless its object is up to date; True if it ran."""
    stamp = obj.with_suffix(".stamp")
    tag = _unit_hash(cmd, src)
    if not force and obj.exists() and stamp.exists() and stamp.read_text() == tag:
        return False
    _run(cmd)
    stamp.write_text(tag)
    return True


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    tag = _sources_hash("v1" + os.environ.get("BKT_BUILD_DIAG", "") + os.environ.get("BKT_BUILD_CROSS", "")
                        + os.environ.get("BKT_BUILD_MARGIN", "") + os.environ.get("BKT_BUILD_DEFS", ""))
    stamp = LIB_DIR / "libbkt.stamp"
    if LIB.exists() and stamp.exists() and stamp.read_text() == tag and not force:
        return LIB
    units: list[tuple[list[str], Path, Path]] = []
    for d in _dims():
        obj = OBJ_DIR / f"leafscan_d{d}.o"
        src = CSRC / "leafscan_inst.cu"
        units.append(([NVCC, *NVFLAGS, f"-DBKT_D={d}", "-c", str(src), "-o", str(obj)], src, obj))
    diag = ["-DBKT_TC_DIAG=1"] if os.environ.get("BKT_BUILD_DIAG") == "1" else []
    if os.environ.get("BKT_BUILD_CROSS") == "1":
        diag.append("-DBKT_TC_CROSS=1")
    if os.environ.get("BKT_BUILD_MARGIN"):
        diag.append(f"-DBKT_TC_MARGIN_LOG2={int(os.environ['BKT_BUILD_MARGIN'])}")
    # experiments: extra -D flags for every CUDA unit, e.g. BKT_BUILD_DEFS="-DBKT_TC_LD4=1"
    diag += [f for f in os.environ.get("BKT_BUILD_DEFS", "").split() if f.startswith("-D")]
    for kt, nr, cps in ((16, 64, 2), (16, 64, 3), (16, 128, 2), (16, 128, 3), (16, 256, 2), (32, 64, 2)):
        for fma in (0, 1):
            obj = OBJ_DIR / f"leafscan_tc_{kt}_{nr}_{cps}_{fma}.o"
            src = CSRC / "leafscan_tc_inst.cu"
            flags = [f"-DBKT_TC_KT={kt}", f"-DBKT_TC_NR={nr}", f"-DBKT_TC_CPS={cps}", f"-DBKT_TC_FMA={fma}", *diag]
            if (kt, nr, cps, fma) == (16, 128, 2, 0):
                flags.append("-DBKT_TC_DISPATCH")
            units.append(([NVCC, *NVFLAGS, *flags, "-c", str(src), "-o", str(obj)], src, obj))
    for name in ("engine.cu", "misc.cu", "build_tree_gpu.cu"):
        obj = OBJ_DIR / (Path(name).stem + ".o")
        src = CSRC / name
        units.append(([NVCC, *NVFLAGS, *diag, "-c", str(src), "-o", str(obj)], src, obj))
    obj = OBJ_DIR / "build_tree.o"
    src = CSRC / "build_tree.cpp"
    units.append((["g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-I", str(INCLUDE), "-c",
                   str(src), "-o", str(obj)], src, obj))
    jobs = jobs or max(1, os.cpu_count() or 1)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        ran = list(ex.map(lambda u: _compile(u[0], u[1], u[2], force), units))
    if verbose:
        print(f"compiled {sum(ran)} of {len(units)} units")
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "--cudart", "static", "-o", str(tmp), *[str(u[2]) for u in units], "-lpthread"])
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
