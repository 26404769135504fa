"""C-ABI library: builds/loads and exports every symbol include/dexel.h declares (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dexel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dexel_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1804_08968_b200 import build as B
    return B.build()


def test_library_exports_every_header_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    syms = header_symbols()
    assert "dexel_dilate" in syms and "dexel_erode" in syms and "dexel_shell" in syms
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath]).decode()
    exported = set(re.findall(r" T (dexel_\w+)", out))
    assert set(syms) <= exported


def test_binding_lists_every_symbol(libpath):
    import paper_1804_08968_b200 as dx
    assert sorted(dx.EXPORTS) == header_symbols()
    L = dx.lib()
    assert L.dexel_last_error() == b""


def test_sm100a_cubin(libpath):
    out = subprocess.check_output(["cuobjdump", "--list-elf", libpath]).decode()
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product path never imports the oracle (independence)."""
    pkg = os.path.join(ROOT, "paper_1804_08968_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "dexel_oracle" not in txt, f


def test_python_api_raises_without_gpu(libpath):
    """No CPU fallback: on a machine without a GPU the ops fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1804_08968_b200 as dx
    with pytest.raises(dx.DexelError):
        dx.Grid(4, 4, -1.0, 1.0)


def test_pipe_suggest_slabs_rule(libpath):
    """dexel_pipe_suggest_slabs is host logic: slabs of >= max(512, 32 R) rows, at most 6, at least 1."""
    import paper_1804_08968_b200 as dx
    f = dx.Pipe.suggest_slabs
    assert f(4096, 4096, 16.0) == 6 and f(2048, 2048, 16.0) == 4 and f(2048, 2048, 64.0) == 1
    assert f(512, 512, 4.0) == 1 and f(64, 64, 3.0) == 1 and f(100000, 100000, 8.0) == 6
    assert f(2048, 2048, 4.0) == 1 and f(2048, 2048, 8.0) == 4      # R < 8: the copies dominate, no split
    assert f(2048, 2048, 16.0, spacing=0.5) == 2          # R = floor(r / s) = 32 -> 1024-row slabs
    for ny in (1, 511, 512, 1023, 1024, 5000):
        for r in (0.0, 0.5, 7.0, 33.0, 255.0):
            s = f(ny, ny, r)
            assert 1 <= s <= 6 and (s == 1 or (r >= 8 and ny // s >= max(512, 32 * int(r))))
