"""The C-ABI library (include/mgrg.h): it loads, exports every declared
symbol, and its host-side validation behaves like the reference's
(errors.hpp codes) -- all without a GPU (no compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2105_12764_b200 import _lib, errors


def declared_functions():
    src = open(_lib.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mgrg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/mgrg.h but not exported"
    assert set(names) == set(_lib.EXPORTS), "EXPORTS list out of sync with the header"


def test_version_and_status_names():
    L = _lib.lib()
    assert b"sm_100a" in L.mgrg_version()
    expect = {1: "InvalidGrid", 2: "InvalidLevel", 3: "ShapeError", 4: "InvalidFusion",
              5: "SingularSystem", 6: "TooManyWorkers", 7: "WorkerFailure",
              8: "CorruptFile", 9: "MissingClass", 10: "InvalidBound", 11: "IoError"}
    for code, name in expect.items():
        assert L.mgrg_status_name(code).decode() == name
        assert errors.from_status(code, "x").code == name


def _create(shape, dtype=4, coords=None, levels=0):
    L = _lib.lib()
    d = _lib.GridDesc()
    d.ndims = len(shape)
    d.dtype = dtype
    for i, s in enumerate(shape):
        d.shape[i] = s
    keep = None
    if coords is not None:
        keep = np.ascontiguousarray(np.concatenate(coords), dtype=np.float64)
        d.coords = keep.ctypes.data
    d.levels = levels
    h = ctypes.c_void_p()
    st = L.mgrg_plan_create(ctypes.byref(d), ctypes.byref(h))
    return st, L.mgrg_last_error().decode()


@pytest.mark.parametrize("shape,coords,code,msg", [
    ((2, 2), None, 1, "no dimension has at least 3 nodes"),
    ((5, 1), None, 1, "need at least 2"),
    ((), None, 1, "1..4 dimensions"),
    ((5,), [np.array([0.0, 1.0, 1.0, 2.0, 3.0])], 1, "not strictly increasing at index 1"),
])
def test_plan_validation_mirrors_reference(shape, coords, code, msg):
    """validate_grid_geometry (grid.cpp:14-36) -> InvalidGrid, before any
    device work."""
    st, what = _create(shape, coords=coords)
    assert st == code
    assert msg in what


def test_plan_rejects_bad_dtype_and_level():
    st, what = _create((9,), dtype=2)
    assert st == 15 and "dtype" in what
    st, what = _create((9,), levels=-1)
    assert st == 2


def test_null_arguments():
    L = _lib.lib()
    assert L.mgrg_plan_create(None, None) == 15
    assert L.mgrg_decompose(None, None, None, None) == 15
    assert L.mgrg_plan_destroy(None) == 0


def test_python_plan_errors_are_reference_types():
    from paper_2105_12764_b200 import Plan

    with pytest.raises(errors.InvalidGrid):
        Plan((2, 2), "float32")
    with pytest.raises(errors.InvalidLevel):
        Plan((9, 9), "float32", levels=0)
    with pytest.raises(errors.InvalidArgument):
        Plan((9,), "int32")


def test_hostio_views_and_copy_pool(tmp_path):
    """The host side of the host-buffer entry points (csrc/hostio.cuh): the
    per-class HostView splits every flat range into exactly the right class
    pieces, and the parallel copy pool copies correctly (no device calls)."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    exe = str(tmp_path / "test_hostio")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(cuda, "include"),
                    os.path.join(root, "tests", "cpp", "test_hostio.cpp"),
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", "-pthread",
                    f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "hostio ok" in out.stdout
