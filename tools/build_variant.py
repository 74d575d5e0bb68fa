"""Build a variant of libautosp.so with extra -D macros for same-box A/B runs
(select it with AUTOSP_LIB=tools/emu/libautosp_<name>.so).

usage: python tools/build_variant.py <name> [-DMACRO=VAL ...]"""

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2604_27089_b200 import _build  # noqa: E402


def main() -> None:
    name, defs = sys.argv[1], sys.argv[2:]
    out_dir = ROOT / "tools" / "emu"
    bdir = out_dir / f"build_{name}"
    bdir.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in _build.SOURCES:
        obj = bdir / (src + ".o")
        subprocess.run([_build.NVCC, *_build.FLAGS, *defs, "-c", str(_build.CSRC / src),
                        "-o", str(obj)], check=True)
        objs.append(str(obj))
    lib = out_dir / f"libautosp_{name}.so"
    subprocess.run([_build.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                    "-o", str(lib), "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
