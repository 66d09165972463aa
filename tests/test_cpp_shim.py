"""The C++ source-level drop-in (include/mgr_b200/refactor.hpp): compiles
against the reference's call shapes here (no GPU), and on a GPU matches the
reference library bit-for-bit (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
PKG = os.path.join(ROOT, "paper_2105_12764_b200")
REF = os.path.join(ROOT, "oracle", "_ref")


def test_header_compiles_standalone():
    subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra",
                    "-I", os.path.join(ROOT, "include"), SRC], check=True)


@pytest.mark.gpu
def test_cpp_shim_matches_reference(tmp_path, oracle_mod):
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    exe = str(tmp_path / "test_shim")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", PKG, "-lmgrg", "-L", REF, "-lmgr_ref", "-pthread",
                    f"-Wl,-rpath,{PKG}:{REF}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "shim ok" in out.stdout


PSRC = os.path.join(ROOT, "tests", "cpp", "test_pipeline_shim.cpp")


def test_pipeline_header_compiles_standalone():
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra",
                    "-I", os.path.join(ROOT, "include"), PSRC], check=True)


@pytest.mark.gpu
def test_cpp_pipeline_shim_matches_reference(tmp_path, oracle_mod):
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    exe = str(tmp_path / "test_pipeline_shim")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), PSRC,
                    "-L", PKG, "-lmgrg", "-L", REF, "-lmgr_ref", "-lz", "-pthread",
                    f"-Wl,-rpath,{PKG}:{REF}", "-o", exe], check=True)
    out = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "pipeline ok" in out.stdout


PARSRC = os.path.join(ROOT, "tests", "cpp", "test_parallel_shim.cpp")


def test_parallel_header_compiles_standalone():
    subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra",
                    "-I", os.path.join(ROOT, "include"), PARSRC], check=True)


@pytest.mark.gpu
def test_cpp_parallel_shim_matches_reference(tmp_path, oracle_mod):
    """cooperative_decompose / grouped_decompose through the C++ drop-in
    (native cooperative runtime) equal the reference's serial decompose."""
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    exe = str(tmp_path / "test_parallel_shim")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), PARSRC,
                    "-L", PKG, "-lmgrg", "-L", REF, "-lmgr_ref", "-pthread",
                    f"-Wl,-rpath,{PKG}:{REF}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "parallel shim ok" in out.stdout


DSRC = os.path.join(ROOT, "tests", "cpp", "test_dropin_contract.cpp")


def test_dropin_contract_compiles_standalone():
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra",
                    "-I", os.path.join(ROOT, "include"), DSRC], check=True)


@pytest.mark.gpu
def test_cpp_dropin_contract_matches_reference(tmp_path, oracle_mod):
    """PassStats (decompose + recompose), weighted_l2_norm, level validation,
    the bounded plan cache, the parallel drivers and CommReport::to_json
    against the reference library."""
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), DSRC,
                    "-L", PKG, "-lmgrg", "-L", REF, "-lmgr_ref", "-lz", "-pthread",
                    f"-Wl,-rpath,{PKG}:{REF}", "-o", exe], check=True)
    out = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    assert "dropin ok" in out.stdout
