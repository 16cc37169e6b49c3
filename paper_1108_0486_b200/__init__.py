"""B200-native xorgensGP (arXiv 1108.0486): sm_100a kernels behind a C ABI.

The product is ``lib/libxg_gpu.so`` (include/xg_gpu.h).  This package is the
Python host mirror of the reference ``xg`` API over it (see ``xorgens.py``).
"""
from .xorgens import *  # noqa: F401,F403
from .xorgens import __all__  # noqa: F401
from . import battery  # noqa: F401,E402  (run_battery_gpu)
