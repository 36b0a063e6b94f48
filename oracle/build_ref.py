"""Stage the reference package in oracle/_ref (TEST / BASELINE INFRASTRUCTURE).

    python oracle/build_ref.py        (also run by __graft_entry__.build())

The reference (``/root/reference/pkg``, pure Python + numba) has no build
step (pkg/pyproject.toml: setuptools, no extension modules), so "building"
it is copying its import package ``pkg/src/csrecon`` unmodified into the
git-ignored ``oracle/_ref/csrecon``.  The copy travels to the GPU box with
the repository snapshot (``oracle/_ref`` is git-ignored, not gpurun-
ignored), where the reference cannot be read; there it is

* the CPU arm of ``bench.py --impl reference`` and ``cpu_baseline``: the
  reference's own ``admm_reconstruct`` with its numba backend on the host
  cores, and
* the host of ``tests/test_reference_binding.py``, which plugs the B200
  kernels into the reference's kernel table and runs the reference's own
  operators and solver against the golden fixtures.

Nothing under ``paper_2006_14080_b200/`` imports it.  ``load()`` imports the
copy with numba's cache redirected to /tmp (the reference JIT-caches with
``cache=True``; the copy must stay unmodified).
"""

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg/src/csrecon"
REF_DIR = os.path.join(HERE, "_ref")


def build(src=REF_PKG, dst=REF_DIR):
    """Copy the reference package into oracle/_ref (no-op without the
    reference, e.g. on the GPU box, where the staged copy is used)."""
    if not os.path.isdir(src):
        return os.path.isdir(os.path.join(dst, "csrecon"))
    target = os.path.join(dst, "csrecon")
    if os.path.isdir(target):
        shutil.rmtree(target)
    os.makedirs(dst, exist_ok=True)
    shutil.copytree(src, target, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    for root, dirs, files in os.walk(target):
        for f in files:
            os.chmod(os.path.join(root, f), 0o644)
    with open(os.path.join(dst, "SOURCE"), "w") as f:
        f.write(f"copied unmodified from {src}\n")
    return True


def available():
    return os.path.isdir(os.path.join(REF_DIR, "csrecon"))


def numba_blas_available():
    """The reference's numba kernels call np.dot inside @njit, which numba
    can only compile with scipy's BLAS bindings present."""
    try:
        from numba.np.linalg import ensure_blas
        ensure_blas()
        return True
    except Exception:
        return False


def load(backend=None):
    """Import the staged reference package (``csrecon``).  backend sets
    CSRECON_BACKEND (kernels.py:32-53) before the import; default: the
    reference's own "auto", or "numpy" where numba cannot compile the
    reference's BLAS calls (no scipy on the host)."""
    if not available():
        raise ImportError("oracle/_ref/csrecon is missing: run oracle/build_ref.py in the "
                          "build container (needs /root/reference)")
    if backend is None:
        backend = "auto" if numba_blas_available() else "numpy"
    os.environ["CSRECON_BACKEND"] = backend
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/csrecon_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import csrecon
    if not os.path.abspath(csrecon.__file__).startswith(REF_DIR):
        raise ImportError(f"csrecon resolved to {csrecon.__file__}, not the staged copy")
    return csrecon


if __name__ == "__main__":
    print("staged" if build() else "reference not found", REF_DIR)
