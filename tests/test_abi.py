"""CPU checks of the C ABI boundary: the library builds/loads and exports every
symbol include/hessketch_b200.h declares; the ctypes table matches the header.
No compute calls (there is no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hessketch_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+|unsigned\s+|long\s+)*\w+\s*\*?\s*(hs_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2502_02721_b200 import _lib, build

    if not build.up_to_date():
        build.build(verbose=False)
    return _lib.LIB_PATH


def test_header_declares_the_boundary():
    names = header_functions()
    for required in ("hs_solve", "hs_op_csr_create", "hs_op_tomo_create", "hs_op_psf_create",
                     "hs_op_dense_create", "hs_sketch_create", "hs_result_trace", "hs_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_header(libpath):
    from paper_2502_02721_b200 import _lib

    assert sorted(_lib.EXPORTED) == header_functions()
    lib = _lib.load()
    assert lib.hs_version().decode().startswith("hessketch_b200")


def test_no_gpu_raises_cleanly(libpath):
    """Without a device every entry point fails loudly (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2502_02721_b200 import _lib

    with pytest.raises(RuntimeError):
        _lib.Context(0)


def test_library_is_sm100a(libpath):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
