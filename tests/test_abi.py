"""CPU-side checks of the boundary: the C-ABI library builds, loads, and exports every symbol
include/cpsgd.h declares (no compute calls -- there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cpsgd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:cp_status|const char\*)\s+(cp_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["cp_sgd_init", "cp_sgd_sample", "cp_sgd_step", "cp_sgd_sweep", "cp_fit", "cp_sgd_destroy"]:
        assert s in syms


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2103_04081_b200 import build

    so = build.build()
    L = ctypes.CDLL(so)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cp_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_binding_covers_every_symbol():
    from paper_2103_04081_b200 import cpsgd

    assert set(declared_symbols()) <= set(cpsgd.EXPORTS)


def test_binding_refuses_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2103_04081_b200 import CPSGD

    X = torch.zeros(24, dtype=torch.float64)
    A = [torch.zeros(2, 1, dtype=torch.float64), torch.zeros(3, 1, dtype=torch.float64),
         torch.zeros(4, 1, dtype=torch.float64)]
    with pytest.raises(ValueError, match="CUDA"):
        CPSGD(X, (2, 3, 4), A, 4)


def test_sass_uses_sm100a():
    """the library carries sm_100a SASS (cuobjdump)."""
    from paper_2103_04081_b200 import build

    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
