"""Build the sm_100a shared library libens.so in-tree (nvcc cross-compiles
without a GPU). Flags: --fmad=false (only the explicit fmas of DESIGN §4 are
fused; the host side likewise with -ffp-contract=off), no fast-math (IEEE
div/sqrt, no FTZ), -lineinfo for ncu source views.

One translation unit per algorithm (csrc/k_*.cu) plus the ABI (csrc/api.cu),
compiled in parallel into csrc/../_obj/*.o (each rebuilt only when a file it
includes changed, from nvcc's -MD dependency lists), then linked."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB = PKG / "libens.so"
OBJ = PKG / "_obj"
CSRC = PKG / "csrc"
UNITS = sorted(CSRC.glob("*.cu"))
SRCS = UNITS + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "ens.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off"]


def nvcc() -> str:
    for c in [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"]:
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _deps(unit: Path) -> list[Path]:
    d = OBJ / (unit.stem + ".d")
    if not d.exists():
        return SRCS
    text = d.read_text().replace("\\\n", " ")
    paths = text.split(":", 1)[1].split() if ":" in text else []
    return [Path(p) for p in paths] or SRCS


def _stale(unit: Path) -> bool:
    o = OBJ / (unit.stem + ".o")
    if not o.exists():
        return True
    t = o.stat().st_mtime
    return any((not p.exists()) or p.stat().st_mtime > t for p in _deps(unit))


def _compile(unit: Path, verbose: bool) -> None:
    o = OBJ / (unit.stem + ".o")
    tmp = o.with_suffix(f".o.tmp{os.getpid()}")
    cmd = [nvcc(), *NVCC_FLAGS, "-MD", "-MF", str(OBJ / (unit.stem + ".d")), "-c", "-o", str(tmp), str(unit)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, o)


def build(force: bool = False, verbose: bool = False) -> Path:
    # a checkout without the object cache (e.g. the snapshot on a GPU box) keeps an up-to-date library
    if not force and not OBJ.exists() and LIB.exists() and LIB.stat().st_mtime >= max(p.stat().st_mtime for p in SRCS):
        return LIB
    OBJ.mkdir(exist_ok=True)
    stamp = OBJ / "flags.txt"
    flags = " ".join([nvcc(), *NVCC_FLAGS])
    if not stamp.exists() or stamp.read_text() != flags:   # compiler or flags changed: rebuild everything
        force = True
    todo = [u for u in UNITS if force or _stale(u)]
    objs = [OBJ / (u.stem + ".o") for u in UNITS]
    if not todo and LIB.exists() and all(LIB.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return LIB
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_compile, u, verbose) for u in todo]:
            f.result()
    tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs)])
    os.replace(tmp, LIB)
    stamp.write_text(flags)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
