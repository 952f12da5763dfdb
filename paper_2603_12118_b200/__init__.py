"""fsx: a B200-native sidecar data plane (Cornserve / fissim hot path).

Layers:
  include/fsx.h + libfsx.so   C ABI: device receive slabs, K1 forward,
                              K3 merge, K0 synth, chunk flags, streaming
                              channels, small-message mailbox (sm_100a)
  include/fsx/fabric.hpp      C++ SidecarFabric-compatible engine
  include/fsx/dropin/fissim   drop-in sidecar.hpp / executor_worker.hpp
  include/fsx/dataplane.hpp   C++ batch pass (forward + merge)
  this package                Python bindings (fabric.py), the batch pass
                              (dataplane.py), traces and shape rules
                              (trace.py), multi-GPU placement (pairs.py,
                              fanout.py) for tests and bench.py
"""
from . import _native, trace  # noqa: F401
from ._native import FsxError  # noqa: F401

__all__ = ["FsxError", "trace", "_native"]
