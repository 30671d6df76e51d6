"""B200-native Tactic decode-time sparse attention (arXiv 2502.12216).

The compute path lives in libtactic.so (hand-written sm_100a CUDA behind the C ABI in
include/tactic.h); `tactic` is its argument-marshalling binding.
"""
from . import tactic  # noqa: F401
from .tactic import (Index, TacticError, build_index, decode, decode_debug, decode_host,  # noqa: F401
                     decode_stage1, decode_stage1b, decode_stage2, dense_decode, device_check,
                     import_index, lse_merge, version)

__version__ = "0.1.0"
