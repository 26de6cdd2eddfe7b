"""Build oracle/_build/liboracle.so from csr_order.c -- TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import pathlib
import subprocess

HERE = pathlib.Path(__file__).resolve().parent
OUT = HERE / "_build" / "liboracle.so"


def build(force: bool = False) -> pathlib.Path:
    src = HERE / "csr_order.c"
    if not force and OUT.exists() and OUT.stat().st_mtime >= src.stat().st_mtime:
        return OUT
    OUT.parent.mkdir(exist_ok=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                    str(src), "-o", str(OUT)], check=True)
    return OUT


REFERENCE_TESTS = pathlib.Path("/root/reference/pkg/tests")
REF_STAGE = HERE / "_ref" / "reftests"
STAGED = ("conftest.py", "test_kernels.py", "test_models.py", "test_selector.py")


def stage_reference_tests() -> pathlib.Path | None:
    """Stage the reference's own kernel / model / selector test files in
    oracle/_ref/reftests (git-ignored; travels to the GPU box like the other
    _ref outputs) so tests/test_dropin_gpu.py can run them unmodified against
    the package.  Only when /root/reference is present (this container)."""
    if not REFERENCE_TESTS.is_dir():
        return REF_STAGE if REF_STAGE.is_dir() else None
    import shutil
    REF_STAGE.mkdir(parents=True, exist_ok=True)
    for name in STAGED:
        shutil.copyfile(REFERENCE_TESTS / name, REF_STAGE / name)
    return REF_STAGE


def load() -> ctypes.CDLL:
    lib = ctypes.CDLL(str(build()))
    P, I64 = ctypes.c_void_p, ctypes.c_int64
    lib.oracle_csr_sum.argtypes = [I64, I64, P, P, P, P, P, P]
    lib.oracle_csr_sum.restype = None
    return lib


def csr_sum(row_ptr, col, val, x):
    """numpy wrapper: reduceat-order CSR sum via the C restatement."""
    import numpy as np
    lib = load()
    V = len(row_ptr) - 1
    x = np.ascontiguousarray(x, np.float32)
    F = x.shape[1]
    y = np.empty((V, F), np.float32)
    rp = np.ascontiguousarray(row_ptr, np.int32)
    c = np.ascontiguousarray(col, np.int32)
    v = None if val is None else np.ascontiguousarray(val, np.float32)
    maxlen = int(np.diff(rp).max()) if V else 0
    scratch = np.empty(max(maxlen, 1) * max(F, 1), np.float32)
    p = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    lib.oracle_csr_sum(V, F, p(rp), p(c), p(v), p(x), p(y), p(scratch))
    return y


if __name__ == "__main__":
    print(build(force=True))
    print(stage_reference_tests())
