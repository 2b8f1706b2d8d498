"""The C-ABI library loads and exports every symbol include/cvb200.h declares;
host-side argument validation answers without launching anything (no GPU)."""

import re
from pathlib import Path

import pytest

from paper_2506_19656_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "cvb200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cv_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    names = declared()
    assert names, "no declarations parsed"
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name


def test_version_and_strings():
    lib = _lib.load()
    assert lib.cv_version() == 100
    assert lib.cv_status_string(0) == b"ok"
    assert lib.cv_max_channels() == 32
    assert lib.cv_num_segments(495, 16) == 31
    assert lib.cv_num_segments(10, 0) == -1
    assert lib.cv_stats_ws_bytes(64, 7) == 64 * 7 * 32


def test_validation_without_launch():
    lib = _lib.load()
    # bad bit depth: rejected before any CUDA call
    st = lib.cv_quantize(1, _lib.CV_F32, 1, 1, 1, 1, 1, 1, 9, 0, 0, 0.0, 16, None, None, None, None,
                         0, 0, 0, 1, None, None, None)
    assert st == _lib.CV_ERR_ARG
    assert b"bit depth 9" in lib.cv_last_error()
    st = lib.cv_stats(1, _lib.CV_F32, 1, 4, 10, 3, 0, 16, 1, None, None, None)
    assert st == _lib.CV_ERR_SHAPE
    st = lib.cv_stats(1, _lib.CV_F32, 1, 4, 66, 33, 0, 16, 1, None, None, None)
    assert st == _lib.CV_ERR_UNSUPPORTED
    st = lib.cv_eval(1, _lib.CV_U16, 3, 1, 1, 10, None, None, 1, _lib.CV_F32, 1, _lib.CV_F32,
                     1, 1, 8, 8, 3, 1, 1, None, 1, 1, 1, None, None)
    assert st == _lib.CV_ERR_ARG  # both frames and recon_in
    st = lib.cv_eval(None, 0, 3, None, None, 8, None, None, 1, _lib.CV_F32, 1, _lib.CV_F32,
                     1, 1, 8, 8, 3, 1, 1, None, 1, 1, 1, None, None)
    assert st == _lib.CV_ERR_SHAPE  # 8x8 frames < 11-px window
    # zero-size work is a no-op success without touching the device
    assert lib.cv_stats_finalize(1, 0, 3, 0, 0.0, None, None, None, None) == _lib.CV_OK
    with pytest.raises(Exception):
        _lib.check(_lib.CV_ERR_ARG, "x")


def test_set_variant_validation():
    """Kernel-variant selection is host-only state: unknown names and CTA sizes
    the launcher has no instantiation for are rejected (gram_nt=128)."""
    lib = _lib.load()
    assert lib.cv_set_variant(b"gram_nt", 128) == _lib.CV_ERR_ARG
    assert b"64 or 256" in lib.cv_last_error()
    assert lib.cv_set_variant(b"no_such_knob", 1) == _lib.CV_ERR_ARG
    for name, default in (("gram_nt", 64), ("gram_tiles", 0), ("proj_nopf", 0), ("qp_px1", 0),
                          ("qp_runtime_c", 0)):
        assert lib.cv_set_variant(name.encode(), default) == _lib.CV_OK
