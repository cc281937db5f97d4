"""B200-native SERE batched-decode MoE path (sm_100a CUDA behind a C-ABI).

Import-light on purpose: the CUDA library (`libsere_b200.so`) is loaded on
first use by :mod:`paper_2602_07616_b200._lib`, and every GPU entry point
raises if it is missing -- there is no CPU fallback.
"""

__version__ = "0.1.0"
