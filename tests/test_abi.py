"""The C-ABI library loads on any host and exports every symbol include/*.h declares."""
import ctypes
import os
import re

from conftest import ROOT


def _declared():
    hdr = open(os.path.join(ROOT, "include", "rsc_b200.h")).read()
    return sorted(set(re.findall(r"\b(rsc_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_header_symbols():
    from paper_1507_05593_b200 import _lib

    assert os.path.exists(_lib.LIB_PATH), "build librsc_b200.so first (__graft_entry__.build())"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == names


def test_version_string_no_gpu_needed():
    from paper_1507_05593_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.rsc_version()


def test_bad_arguments_rejected_without_gpu():
    from paper_1507_05593_b200 import _lib

    lib = _lib.load()
    assert lib.rsc_gemm_grouped(0, 0, None, -1, None) < 0
    assert lib.rsc_potrf_batched(-1, None, None, None, None, None, None) < 0
    assert lib.rsc_trsm_batched(5, 0, 1, None, None, None, None, None, None, None, None) < 0
    assert lib.rsc_qrcp_batched(-1, None, None, None, None, None, None, None, None, None) < 0


def test_gemm_descriptor_layout_matches_header():
    from paper_1507_05593_b200._lib import GEMM_DTYPE

    assert GEMM_DTYPE.itemsize == 128
    assert GEMM_DTYPE.fields["alpha"][1] == 104
    assert GEMM_DTYPE.fields["ext_r"][1] == 120
