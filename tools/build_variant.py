#!/usr/bin/env python
"""Build an experimental variant of libens.so for A/B timing (never the product).

  python tools/build_variant.py NAME UNIT[,UNIT...] [-DMACRO=VALUE ...]

Compiles the listed translation units (e.g. k_ros23) with the extra macros into
paper_2304_06835_b200/_variants/NAME/, links them with the product's objects of
every other unit (paper_2304_06835_b200/_obj, built first), and writes
_variants/NAME/libens.so. tools/ab_variants.py loads each variant in its own
process (by pointing the binding's _LIB_PATH at it) and times the same configs."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2304_06835_b200 import _build  # noqa: E402


def main():
    name, units = sys.argv[1], sys.argv[2].split(",")
    defs = [a for a in sys.argv[3:] if a.startswith("-D")]
    _build.build()
    out = _build.PKG / "_variants" / name
    out.mkdir(parents=True, exist_ok=True)
    objs = []
    todo = []
    for u in _build.UNITS:
        if u.stem in units:
            o = out / (u.stem + ".o")
            todo.append([_build.nvcc(), *_build.NVCC_FLAGS, *defs, "-c", "-o", str(o), str(u)])
            objs.append(o)
        else:
            objs.append(_build.OBJ / (u.stem + ".o"))
    with ThreadPoolExecutor(len(todo) or 1) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in todo]:
            f.result()
    subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "-o", str(out / "libens.so"), *map(str, objs)])
    (out / "defs.txt").write_text(" ".join(defs) + "\n")
    print(out / "libens.so")


if __name__ == "__main__":
    main()
