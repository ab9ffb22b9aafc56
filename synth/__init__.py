"""Seeded synthetic inputs shared by tests and bench (no attention arithmetic here).

The paper draws Q, K, V from U[0,1).  For reproducibility across CPU and
GPU every element is a pure function of (seed, tensor, flat index) — reading R22:

    u = splitmix64(splitmix64(seed + tau) XOR e),   tau = 0 (Q), 1 (K), 2 (V)
    e = (token * H + head) * d + c
    x = (u >> 40) * 2^-24  in [0, 1), exact in fp32, then RNE to bf16 / fp16.

splitmix64(x) is the SplitMix64 output function of state x + 0x9e3779b97f4a7c15.
Three independent implementations exist (this NumPy one, oracle.c's, and the CUDA
ga_fill_inputs kernel); tests/golden/rng.txt pins all three.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GAMMA = 0x9E3779B97F4A7C15


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix64(x: int) -> int:
    return int(splitmix64_np(np.array([x & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


def uniform_f32(seed: int, tensor: int, n: int, e0: int = 0) -> np.ndarray:
    """n consecutive fp32 values of tensor `tensor`, starting at flat index e0."""
    base = np.uint64(splitmix64((seed + tensor) & 0xFFFFFFFFFFFFFFFF))
    e = np.arange(e0, e0 + n, dtype=np.uint64)
    u = splitmix64_np(base ^ e)
    return (u >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)


def qkv(seed: int, L: int, H: int, d: int, dtype: str = "f32", centred: bool = False):
    """Seeded (Q, K, V) as torch CPU tensors [L, H, d] in the storage dtype.

    centred=True subtracts 0.5 in fp32 before rounding (the parity-stress variant of
    SURVEY §8(d)); it is exact in fp32 for these values.
    """
    import torch

    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dtype]
    out = []
    for t in range(3):
        a = uniform_f32(seed, t, L * H * d)
        if centred:
            a = a - np.float32(0.5)
        out.append(torch.from_numpy(a.reshape(L, H, d)).to(tdt))  # torch .to() is RNE
    return tuple(out)


def as_f64(t) -> np.ndarray:
    """Exact fp64 copy of a stored tensor (bf16/fp16/fp32 -> fp64 is exact)."""
    return t.double().numpy()
