"""B200-native graph-view masked attention (arXiv 2502.01659, "Longer Attention Span").

Thin Python binding over libga.so (include/ga.h).  Tokens are graph nodes, mask nonzeros
are edges; one fused CUDA pass per row computes q.k/sqrt(d), an online softmax over the
row's neighbours and the weighted sum of their values (Algorithm 1).
"""
from .attention import (GraphAttention, State, attention, attention_backward, attention_host, compose, coo_to_csr, fill_inputs, mask_count, mask_to_csr,
                        mask_validate, qkv_device, query_alignment, state_finalize, version, workspace_size)
from .masks import BB_GLOBAL, BB_RANDOM, BB_WINDOW, CSR, BigBird, BlockDilated, LongNet, Mask, Window
from . import presets
from ._abi import GaError

__all__ = ["attention", "attention_backward", "GraphAttention", "attention_host", "compose", "coo_to_csr", "fill_inputs", "mask_count", "mask_to_csr", "mask_validate",
           "qkv_device", "query_alignment", "state_finalize", "version", "workspace_size", "State", "CSR", "BigBird",
           "BlockDilated", "LongNet", "Mask", "Window", "BB_WINDOW", "BB_GLOBAL", "BB_RANDOM", "presets", "GaError"]
