"""Build libcsrecon_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2006_14080_b200.build [-v]

The library is a plain C-ABI shared object (no torch types) linked against
the NCCL that ships with torch (site-packages/nvidia/nccl), so the process
loads exactly one libnccl.
"""

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libcsrecon_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root():
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")]
    try:
        import nvidia  # noqa: F401
        cands += [os.path.join(p, "nccl") for p in nvidia.__path__]
    except ImportError:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (expected torch's nvidia-nccl package)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(REPO, "include", "*.h")))


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False, defines=(), out=None):
    """Compile the library; `defines`/`out` build a profiling variant
    (tools/build_variants.py) instead of the product library."""
    if out is None and not defines and not force and up_to_date():
        return OUT
    out = out or OUT
    nccl = nccl_root()
    cmd = (["nvcc"] + ARCH + [f"-D{d}" for d in defines] +
           ["-O3", "-lineinfo", "-std=c++17", "-shared",
                              "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                              "-I", os.path.join(nccl, "include"),
                              "-I", os.path.join(REPO, "include"),
                              os.path.join(CSRC, "csrecon_b200.cu"),
                              "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                              "-Xlinker", "-rpath," + os.path.join(nccl, "lib"),
                              "-o", out + ".tmp"])
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode:
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    os.replace(out + ".tmp", out)
    with open(out[:-3] + ".ptxas.log" if out != OUT else os.path.join(HERE, "ptxas.log"),
              "w") as f:
        f.write(res.stderr)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
