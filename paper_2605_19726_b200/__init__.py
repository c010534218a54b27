"""B200-native (sm_100a) hot path of BA-Att (arXiv 2605.19726).

The product is libbaatt.so (C ABI, include/ba_attn.h); ``baatt`` is its thin
Python binding.  This package never imports the CPU oracle.
"""
from .baatt import (BaError, Context, Selection, ba_attention, ba_attention_host, ba_dense_attn,  # noqa: F401
                    ba_select, ba_sparse_attn, load)
