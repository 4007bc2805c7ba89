"""B200-native (sm_100a) ChunkFT chunk-local training step.

Host planning (partitioner, plan hash, rotation scheduler) and all compute live in the
native library libchunkft_b200.so behind the C ABI in include/chunkft_b200.h; this package
is the Python-side mirror of the reference's operator API (include/chunkft/*.hpp).
"""
from . import _native  # noqa: F401  (raises ImportError if the native library is missing)

__all__ = ["_native"]
