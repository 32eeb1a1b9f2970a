"""CPU-side checks of the C ABI library and host logic (no kernel launches)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2504_21719_b200 import _abi, _native
from paper_2504_21719_b200.errors import NativeUnavailable
from paper_2504_21719_b200.radiomap import MeasurementGrid, RadioMapConfig


def _header_functions():
    text = open(os.path.join(ROOT, "include", "sbr.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sbr_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _native.load_library()
    declared = _header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/sbr.h but not exported"
    assert set(_native.exported_symbols()) <= set(declared)
    assert lib.sbr_version() >= 100


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_struct_layouts_match_header():
    # SbrMaterial: 10 doubles + 4 int32 = 96 bytes; SbrAntenna: 2 int32 + 10 doubles
    assert ctypes.sizeof(_abi.SbrMaterial) == 96
    assert ctypes.sizeof(_abi.SbrAntenna) == 88
    assert ctypes.sizeof(_abi.SbrMapParams) % 8 == 0


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(NativeUnavailable):
        _native.lib()


def test_error_status_mapping():
    _native.load_library()
    from paper_2504_21719_b200.errors import EmptyScene
    with pytest.raises(EmptyScene):
        _native.check(_abi.SBR_ERR_EMPTY_SCENE)
    with pytest.raises(ValueError):
        _native.check(_abi.SBR_ERR_INVALID)
    with pytest.raises(RuntimeError):
        _native.check(_abi.SBR_ERR_STACK)


def test_grid_geometry_and_validation():
    g = MeasurementGrid((1.0, 2.0, 3.0), (1, 0, 0), (0, 1, 0), (0.5, 0.25), (4, 8))
    assert np.allclose(g.normal, [0, 0, 1])
    assert g.cell_area == pytest.approx(0.125)
    assert np.allclose(g.corner, [0.0, 1.0, 3.0])
    assert g.cell_centers().shape == (8, 4, 3)
    h = MeasurementGrid.horizontal((0, 0, 1.5), (10.0, 6.0), (2.0, 2.0))
    assert h.shape == (5, 3)
    lookup = MeasurementGrid((0.0, 0.0, 2.0), (1, 0, 0), (0, 1, 0), (1.0, 1.0), (2, 2))
    assert lookup.cell_lookup((0.0, 0.0, 2.0)) == (1, 1)
    assert lookup.cell_lookup((1.001, 0.0, 2.0)) is None
    with pytest.raises(ValueError, match="unit"):
        MeasurementGrid((0, 0, 0), (2, 0, 0), (0, 1, 0), (1, 1), (2, 2))
    with pytest.raises(ValueError, match="orthogonal"):
        MeasurementGrid((0, 0, 0), (1, 0, 0), (1, 0, 0), (1, 1), (2, 2))


def test_config_validation():
    with pytest.raises(ValueError):
        RadioMapConfig(num_samples=0)
    with pytest.raises(ValueError):
        RadioMapConfig(rr_max=0.0)
    with pytest.raises(ValueError):
        RadioMapConfig(rr_depth=4, max_depth=3)
    with pytest.raises(ValueError):
        RadioMapConfig(gain_threshold=-1.0)
    assert RadioMapConfig().wavelength == pytest.approx(299792458.0 / 3.5e9)


def test_exact_maps_switch_checked():
    """sbr_set_exact_maps takes 0 / 1 (pure host setter, no device call)."""
    lib = _native.load_library()
    assert lib.sbr_set_exact_maps(2) == _abi.SBR_ERR_INVALID
    assert lib.sbr_set_exact_maps(-1) == _abi.SBR_ERR_INVALID
    assert lib.sbr_set_exact_maps(1) == 0 and lib.sbr_set_exact_maps(0) == 0


def test_wave_streams_range_checked():
    """sbr_set_wave_streams accepts 1..4 (pure host setter, no device call)."""
    lib = _native.load_library()
    assert lib.sbr_set_wave_streams(0) == _abi.SBR_ERR_INVALID
    assert lib.sbr_set_wave_streams(5) == _abi.SBR_ERR_INVALID
    assert lib.sbr_set_wave_streams(2) == 0
