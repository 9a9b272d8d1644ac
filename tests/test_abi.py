"""The C-ABI library loads and exports every function include/latham_b200.h declares (CPU only:
no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "latham_b200.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lt_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1408_3839_b200 import native
    if not os.path.exists(native.LIB_PATH):
        subprocess.run(["make", "-j8"], cwd=os.path.join(ROOT, "paper_1408_3839_b200", "csrc"), check=True,
                       capture_output=True)
    return ctypes.CDLL(native.LIB_PATH)


def test_every_declared_symbol_is_exported(lib):
    names = declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_1408_3839_b200 import native
    assert sorted(native.EXPORTS) == declared()


def test_sm100a_code_in_library(lib):
    from paper_1408_3839_b200 import native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_device(lib):
    # with no CUDA device the product raises instead of computing on the host
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1408_3839_b200.api import Context
    with pytest.raises(Exception):
        Context(0)
