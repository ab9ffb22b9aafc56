"""B200-native graph-view masked attention (arXiv 2502.01659, "Longer Attention Span").

Thin Python binding over libga.so (include/ga.h).  Tokens are graph nodes, mask nonzeros
are edges; one fused CUDA pass per row computes q.k/sqrt(d), an online softmax over the
row's neighbours and the weighted sum of their values (Algorithm 1).
"""
from .attention import (attention, attention_host, fill_inputs, mask_count, mask_to_csr, mask_validate,
                        qkv_device, query_alignment, version, workspace_size)
from .masks import CSR, BigBird, BlockDilated, LongNet, Mask, Window
from ._abi import GaError

__all__ = ["attention", "attention_host", "fill_inputs", "mask_count", "mask_to_csr", "mask_validate",
           "qkv_device", "query_alignment", "version", "workspace_size", "CSR", "BigBird", "BlockDilated", "LongNet", "Mask",
           "Window", "GaError"]
