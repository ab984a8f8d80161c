"""B200-native TiMePReSt pipeline-parallel training step.

Python mirror of the reference's ``pipesim`` API (proj/include/pipesim/*.hpp)
over the C ABI in ``include/pipesim_b200.h``.  The compute path is the
sm_100a library in ``lib/``; there is no CPU fallback.
"""
from ._native import (CapacityError, CudaError, DomainError,  # noqa: F401
                      InsufficientHorizonError, IntegrityError, IoError,
                      PipesimError, StructuralError)

__all__ = [
    "PipesimError", "DomainError", "StructuralError", "InsufficientHorizonError",
    "IntegrityError", "IoError", "CudaError", "CapacityError",
]
