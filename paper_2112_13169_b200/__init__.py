"""B200-native per-frame voxelization (arXiv 2112.13169) behind the reference
voxmap API. Product code: csrc/ (sm_100a kernels + C-ABI), _native.py (ctypes
binding of include/vxm.h) and voxmap.py (Python mirror of the reference API).
The C++ drop-in headers live in include/voxmap/."""

__all__ = ["voxmap"]
