"""Build profiling variants of the native library with extra -D flags, in
parallel: python tools/build_variants.py name1=DEF_A=1,DEF_B=0 name2=...
Load one with CSR_VARIANT=name (paper_2006_14080_b200/variants/name.so)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_14080_b200 import build

VDIR = os.path.join(build.HERE, "variants")


def one(spec):
    name, _, defs = spec.partition("=")
    defines = [d for d in defs.split(",") if d]
    out = os.path.join(VDIR, name + ".so")
    build.build(defines=defines, out=out)
    return name


if __name__ == "__main__":
    os.makedirs(VDIR, exist_ok=True)
    with ThreadPoolExecutor(len(sys.argv) - 1) as ex:
        for n in ex.map(one, sys.argv[1:]):
            print("built", n)
