"""fsx: a B200-native sidecar data plane (Cornserve / fissim hot path).

Layers:
  include/fsx.h + libfsx.so   C ABI: device receive slabs, K1 forward,
                              K3 merge, K0 synth, chunk flags (sm_100a)
  include/fsx/fabric.hpp      C++ SidecarFabric-compatible engine (drop-in)
  this package                Python bindings for tests and bench
"""
from . import _native, trace  # noqa: F401
from ._native import FsxError  # noqa: F401

__all__ = ["FsxError", "trace", "_native"]
