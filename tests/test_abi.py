"""The C-ABI boundary: the shared library loads and exports every entry point
include/cdg_gpu.h declares (no compute calls: this runs without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_1208_4772_b200 import gpu

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "cdg_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(cdg_gpu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("cdg_gpu_level_create", "cdg_gpu_compute_rhs", "cdg_gpu_rk_steps", "cdg_gpu_interpolate_to_faces",
              "cdg_gpu_viscosity", "cdg_gpu_aux_gradient", "cdg_gpu_timestep", "cdg_gpu_residual"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(gpu.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_version_string():
    assert b"sm_100a" in gpu.lib().cdg_gpu_version()


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the product fails loudly (status 4)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1208_4772_b200 import mesh
    with pytest.raises(gpu.CudaError):
        gpu.GpuLevel(mesh.cube_mesh(1), 2)


def test_config_errors_are_config_errors():
    with pytest.raises(gpu.ConfigError):
        gpu.run_config("roe")
