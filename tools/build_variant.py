"""Build a variant of libdfx.so for kernel sweeps (benchmarking only): every csrc/*.cu compiled with extra
-D flags (and optionally a replacement source for one file) into DIR/libdfx.so; select it at run time with
DFX_LIB_PATH=DIR/libdfx.so. The product build is paper_2507_13833_b200/build.py.

usage: python tools/build_variant.py DIR [-D NAME=VALUE ...] [--replace loss.cu=/path/to/other.cu]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import importlib.util
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_dfx_build", os.path.join(ROOT, "paper_2507_13833_b200", "build.py"))
B = importlib.util.module_from_spec(spec)
spec.loader.exec_module(B)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("-D", action="append", default=[])
    ap.add_argument("--replace", action="append", default=[])
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    repl = dict(r.split("=", 1) for r in a.replace)
    defs = [f"-D{d}" for d in a.D]

    def comp(src):
        name = os.path.basename(src)
        real = os.path.abspath(repl.get(name, src))
        obj = os.path.join(a.out, name.replace(".cu", ".o"))
        cmd = [B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, f"-I{B.CSRC}", *defs, "-c", real, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, B.sources()))
    lib = os.path.join(a.out, "libdfx.so")
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-ldl"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
