"""CPU-side checks of the C ABI boundary: the library builds, loads, and
exports every symbol include/pacim.h declares; calls fail loudly (no CPU
fallback) when no GPU is present."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pacim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pacim_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2311_07554_b200 import build
    return build.build()


def test_header_lists_boundary_calls():
    syms = header_symbols()
    for s in ["pacim_load_graph", "pacim_build_sketches", "pacim_select_seeds"]:
        assert s in syms


def test_library_exports_every_header_symbol(libpath):
    L = ctypes.CDLL(libpath)
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_binding_names_match_header(libpath):
    from paper_2311_07554_b200 import binding
    assert sorted(binding.EXPORTS) == header_symbols()
    for s in header_symbols():
        if s in ("pacim_create", "pacim_destroy", "pacim_last_error", "pacim_version",
                 "pacim_threshold_from_p", "pacim_threshold_uniform", "pacim_nccl_unique_id"):
            continue
        assert hasattr(binding.Context, s), s


def test_threshold_from_p_host_only(libpath):
    from paper_2311_07554_b200 import pacim_threshold_from_p
    assert pacim_threshold_from_p(0.0) == 0
    assert pacim_threshold_from_p(0.5) == 1 << 31
    assert pacim_threshold_from_p(1.0) == 1 << 32
    assert pacim_threshold_from_p(0.02) == 85899345


def test_no_gpu_fails_loudly(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2311_07554_b200 import Context, PacimError
    with pytest.raises(PacimError):
        Context(0)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2311_07554_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower(), f


def test_nccl_linked_in_library(libpath):
    """The multi-GPU path calls NCCL from the library (dist.cu): libpacim.so
    depends on libnccl.so.2 (the venv's build, the one torch loads)."""
    import subprocess
    out = subprocess.run(["ldd", libpath], capture_output=True, text=True).stdout
    assert "libnccl.so.2" in out
