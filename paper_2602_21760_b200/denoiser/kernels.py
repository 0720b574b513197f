"""ctypes bindings of the denoiser kernels (include/hybridpar_b200_denoiser.h)."""
from __future__ import annotations

from .. import _native as N

SIGNATURES: dict = {}
N.register_signatures(SIGNATURES)
