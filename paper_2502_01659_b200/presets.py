"""The paper's Fig. 5 mask presets as disjoint components + their union.

"For all approaches the local size was set to 50 in each direction and three global tokens
were used, the dilated local window used a dilation factor of two giving an effective local
size of 100, and S_f = 0.001 for the random sparsity".  Under reading R2 a
local size of n each way is Window(n + 1); the dilated window is Window(2n + 1, r = 2) (50
neighbours each way, 100 tokens apart at most); S_f = 0.001 is 0.001 L random columns per
non-global row (reading R10).

Each preset returns the components the paper runs as sequential kernel calls (local, the
global kernel = "global minus local", random) — disjoint, so
`compose(q, k, v, components)` carries one state through them — and the union as one
explicit CSR (the paper's single-CSR variant).  Non-window components are materialised as
device CSR with ga_mask_to_csr.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

from .attention import mask_to_csr
from .masks import BB_GLOBAL, BB_RANDOM, BigBird, Mask, Window

PAPER_LOCAL = 50      # tokens in each direction
PAPER_GLOBALS = 3     # global tokens
PAPER_DILATION = 2    # dilated Longformer
PAPER_SF = 1e-3       # random sparsity of BigBird


@dataclass
class Preset:
    name: str
    components: List[Mask]  # disjoint; Window implicit, the rest device CSR
    union: Mask             # one explicit CSR of the whole pattern
    pattern: BigBird        # the implicit descriptor the union was generated from


def _build(name, L, w, r, n_global, n_random, seed, parts_list) -> Preset:
    full = BigBird(w, n_global, n_random, seed=seed, r=r)
    comps: List[Mask] = [Window(w, r)]
    for parts in parts_list:
        comps.append(mask_to_csr(BigBird(w, n_global, n_random, seed=seed, r=r, parts=parts), L))
    return Preset(name, comps, mask_to_csr(full, L), full)


def longformer(L: int, local: int = PAPER_LOCAL, n_global: int = PAPER_GLOBALS) -> Preset:
    """Fig. 5 left: local (n each way) + global tokens."""
    return _build("longformer", L, local + 1, 1, n_global, 0, 0, [BB_GLOBAL])


def longformer_dilated(L: int, local: int = PAPER_LOCAL, dilation: int = PAPER_DILATION,
                       n_global: int = PAPER_GLOBALS) -> Preset:
    """Fig. 5 middle: dilated local window (n neighbours each way, `dilation` apart) + globals."""
    return _build("longformer_dilated", L, local * dilation + 1, dilation, n_global, 0, 0, [BB_GLOBAL])


def bigbird(L: int, local: int = PAPER_LOCAL, n_global: int = PAPER_GLOBALS, s_f: float = PAPER_SF,
            seed: int = 0xB16B12D) -> Preset:
    """Fig. 5 right: local + global + random (S_f L random columns per non-global row)."""
    n_random = max(1, int(round(s_f * L)))
    return _build("bigbird", L, local + 1, 1, n_global, n_random, seed, [BB_GLOBAL, BB_RANDOM])
