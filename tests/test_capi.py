"""CPU-side checks of the C ABI: the library loads and exports every symbol the
header declares (no compute calls: there is no GPU here)."""

import ctypes
import os
import re

import pytest

from paper_1801_02362_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    with open(os.path.join(ROOT, "include", "mcb200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^(?:int|int64_t)\s+(mc_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for name in ("mc_center", "mc_cov_f64", "mc_fit_dense", "mc_fit_full", "mc_rot_grad", "mc_close_scan",
                 "mc_pathcv_weights", "mc_pathcv_grad", "mc_pair_grad", "mc_property_map"):
        assert name in syms


def test_library_loads_and_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmcb200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.mc_version() == 1
    # every binding the Python shim declares is in the header too
    assert set(_lib.exported_symbols()) <= set(header_symbols()) | {"mc_version"}


def test_status_mapping_raises_reference_errors():
    from paper_1801_02362_b200 import errors

    _lib.check(0)
    for code, cls in ((-1, errors.InvalidStructureError), (-2, errors.DegenerateFitError), (-3, errors.ConfigError),
                      (-5, errors.EmptyActiveSetError), (-102, errors.DeviceError)):
        with pytest.raises(cls):
            _lib.check(code, "x")


def test_argument_validation_without_gpu():
    """Validation happens before any launch: bad arguments return status codes on a CPU box."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmcb200.so not built")
    lib = _lib.load()
    # n < 2 -> InvalidStructure; npad not a multiple of 32 -> Config
    assert lib.mc_center(None, 1, 0, 1, 32, None, None, None, None, None, None, None, None, None, None) == -1
    assert lib.mc_center(None, 1, 0, 5, 33, None, None, None, None, None, None, None, None, None, None) == -3
    assert lib.mc_property_map(0, 0, None, None, None, 1.0, None, None, None, None) == -5
    assert lib.mc_close_scan(None, None, 1, 1, 32, None, None, 0, 0.1, None, None, None, None, None) == -3
