"""Rotary frequency tables for the retrieval head's front-end (spc_rethead_qk) — host setup.

Paper §4.3: the 2k-context DLM is extended to long contexts "using the training-free
method provided by YaRN".  YaRN ("NTK-by-parts" interpolation, Peng et al. 2023) rescales each
rotary frequency by how many of its wavelengths fit in the original context:
    theta_i = base^(-2i/D),  lambda_i = 2 pi / theta_i,  r_i = L_orig / lambda_i,
    gamma_i = clamp((r_i - beta_slow) / (beta_fast - beta_slow), 0, 1),
    theta'_i = (1 - gamma_i) * theta_i / s + gamma_i * theta_i,
so wavelengths that fit fewer than beta_slow times are interpolated by the full factor s,
those that fit more than beta_fast times are kept, and the band between is blended; the
attention scale ("temperature") is mscale = 0.1 ln(s) + 1 for s > 1, applied to cos and sin
(so q.k scales by mscale^2).  This is a one-time table computation (not per-step work): the
per-step rotation runs in libspc.  Reading R24 in DESIGN.md.
"""
from __future__ import annotations

import math

import numpy as np


def yarn_inv_freq(D: int, base: float = 500000.0, factor: float = 1.0, orig_ctx: int = 2048,
                  beta_fast: float = 32.0, beta_slow: float = 1.0):
    """(inv_freq [D/2] float32, mscale float) for head dim D (factor 1: plain RoPE)."""
    i = np.arange(D // 2, dtype=np.float64)
    theta = base ** (-2.0 * i / D)
    if factor <= 1.0:
        return theta.astype(np.float32), 1.0
    r = orig_ctx * theta / (2.0 * math.pi)  # wavelengths of dim i that fit in the context
    gamma = np.clip((r - beta_slow) / (beta_fast - beta_slow), 0.0, 1.0)
    inv = (1.0 - gamma) * theta / factor + gamma * theta
    return inv.astype(np.float32), 0.1 * math.log(factor) + 1.0
