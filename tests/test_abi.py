"""C-ABI boundary checks that need no GPU: the library builds/loads, exports every symbol
include/akmc.h declares, and fails loudly (no CPU fallback) when no CUDA device exists."""
import ctypes

import numpy as np
import pytest

import paper_2604_24091_b200 as akmc
from paper_2604_24091_b200 import build


def test_library_exports_header_symbols():
    build.build()
    lib = akmc.load()
    syms = akmc.header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.akmc_version().startswith(b"akmc-b200")


def test_struct_layout_matches_header():
    # akmc_config: 3+1+1+1+1+3 int32 (40 B) + pad to 8 + 4 doubles + u64 + 3+2 int32
    assert ctypes.sizeof(akmc.akmc.CConfig) == 40 + 32 + 8 + 20 + 128 + 4
    assert ctypes.sizeof(akmc.akmc.CCounters) == 9 * 8 + 2 * 8


def test_invalid_config_rejected_before_device():
    lib = akmc.load()
    bad = akmc.Config(cells=(7, 8, 8))
    with pytest.raises(akmc.AkmcError) as e:
        akmc.Simulation(bad, np.zeros(2 * 7 * 64, np.uint8), np.zeros((2, 7, 7)), np.zeros(7))
    assert e.value.code == akmc.AKMC_ERR_INVALID
    eps = np.zeros((2, 7, 7)); eps[0, 1, 2] = 1.0       # asymmetric
    with pytest.raises(akmc.AkmcError) as e:
        akmc.Simulation(akmc.Config(cells=(4, 4, 4)), np.zeros(128, np.uint8), eps, np.zeros(7))
    assert e.value.code == akmc.AKMC_ERR_INVALID
    with pytest.raises(akmc.AkmcError) as e:
        akmc.Simulation(akmc.Config(cells=(16, 16, 16), domain_cells=(4, 4, 4), window_s=1.0),
                        np.zeros(8192, np.uint8), np.zeros((2, 7, 7)), np.zeros(7))
    assert e.value.code == akmc.AKMC_ERR_INVALID


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(akmc.AkmcError) as e:
        akmc.Simulation(akmc.Config(cells=(4, 4, 4)), np.zeros(128, np.uint8), np.zeros((2, 7, 7)), np.zeros(7))
    assert e.value.code == akmc.AKMC_ERR_CUDA


def test_entry_points_reject_bad_arguments_without_device():
    """Argument checks of the newer entry points happen before any device work (header contracts)."""
    lib = akmc.load()
    x = np.zeros(4)
    y = np.zeros(4)
    p = ctypes.c_void_p
    assert lib.akmc_debug_math(7, p(x.ctypes.data), 4, p(y.ctypes.data)) == akmc.AKMC_ERR_INVALID   # unknown fn
    assert lib.akmc_debug_math(0, None, 4, p(y.ctypes.data)) == akmc.AKMC_ERR_INVALID
    assert lib.akmc_debug_math(0, None, 0, None) == akmc.AKMC_OK                                    # empty batch
    ctr = akmc.akmc.CCounters()
    assert lib.akmc_run_until(None, 1.0, 10, ctypes.byref(ctr)) == 1                                 # AKMC_ERR_RUNTIME
    assert lib.akmc_set_voxel_temperatures(None, p(x.ctypes.data), 4) == 1
    assert lib.akmc_step(None, 1, ctypes.byref(ctr)) == 1


def test_no_device_math_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(akmc.AkmcError) as e:
        akmc.debug_math(0, np.zeros(8))
    assert e.value.code == akmc.AKMC_ERR_CUDA
