"""B200-native (sm_100a) constant-pH lambda-dynamics step library (arXiv 2410.01626).

The compute path is libcph.so (hand-written CUDA kernels + cuFFT) behind the C ABI
in include/cph.h; `binding` marshals numpy arrays into it; `titration` gathers
lambda frames across ranks (NCCL via torch.distributed) and fits
Henderson-Hasselbalch / Hill curves on the host.
"""
from .binding import (CphError, Context, ENERGY_TERMS, KERNEL_CLASSES, cph_create,  # noqa: F401
                      lib, load_library)
_lib_handle = lib()   # load now: no silent CPU fallback
