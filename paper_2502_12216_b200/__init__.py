"""B200-native Tactic decode-time sparse attention (arXiv 2502.12216).

The compute path lives in libtactic.so (hand-written sm_100a CUDA behind the C ABI in
include/tactic.h); `tactic` is its argument-marshalling binding.
"""
from . import tactic  # noqa: F401
from .tactic import (DecodeSession, Index, TacticError, append, assign_tokens, build_index, decode,  # noqa: F401
                     decode_attention_only, decode_debug, decode_fixed_budget, decode_host, decode_per_head, decode_stage1,
                     decode_stage1b, decode_stage2, dense_decode, device_check, exact_logits, import_index,
                     lse_merge, set_options, set_tail_capacity, tail_info, version)

__version__ = "0.1.0"
