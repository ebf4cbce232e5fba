"""B200-native sparse-inverse local-global solver with non-smooth frictional
contact (arXiv 2503.15078).  Thin ctypes binding over the C ABI in
include/sim.h; every step of the hot path runs in libsim.so's CUDA kernels.
There is no CPU fallback: if libsim.so is missing or has no device, calls fail.
"""
from ._lib import (Sim, SimError, lib, lib_path, MODEL_NEOHOOKEAN, MODEL_COROTATED,  # noqa: F401
                   MODEL_ARAP, EXPORTED_SYMBOLS, KERNEL_KINDS, CONTACT_DTYPE, contacts_to_array,
                   use_torch_allocator)

__all__ = ["Sim", "SimError", "lib", "lib_path", "EXPORTED_SYMBOLS"]
