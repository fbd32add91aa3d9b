"""distwar-b200: B200-native DISTWAR (arXiv 2401.05345) hot path.

The product is ``csrc/libdistwar.so`` (CUDA for sm_100a behind the C ABI in
``include/distwar.h``); this package is the host-side mirror of the
reference's interface over that ABI:

* ``warpred``    -- traces, policies, GPU reduction, threshold tuning
* ``rasterizer`` -- render_forward / render_backward of a Gaussian-splatting
                    view with the DISTWAR backward
* ``scene``      -- synthetic scenes and cameras of the BASELINE configs
* ``dist``       -- view-parallel backward + gradient all-reduce
"""
from ._lib import DistwarError, InvalidArgument, IOFailure, LIB_PATH, lib  # noqa: F401

__version__ = "0.1.0"
