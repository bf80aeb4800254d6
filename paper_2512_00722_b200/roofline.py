"""Roofline accounting for the hot path (host arithmetic only).

Algorithmic bytes of one decode step, per request b:
    retrieval keys   S_b * G * D * e            (spc_score streams every key once)
  + selected K and V L * G * min(k, S_b) * D * e * 2   (spc_sparse_decode_attn)
e = bytes per element (2 for bf16).  Queries, indices, logits, scores and
outputs are overhead, not counted.  The KV-footprint formula this rests on is
pinned to the paper's anchors (2 GB at 16K; 4 GB at 32K for
Llama3.1-8B) in tests/test_roofline.py.
"""
from __future__ import annotations


def kv_bytes(L: int, H: int, D: int, S: int, bytes_per_elem: int = 2) -> int:
    """Dense KV-cache bytes: K and V, L layers, H KV heads, S tokens."""
    return 2 * L * H * D * S * bytes_per_elem


def retrieval_overhead(layers: int, bsz: int, heads: int, dim: int, len_keys: int,
                       o_mul: int = 1) -> int:
    """Eq.3: O_tot = layers * bsz * heads * dim * len_keys * O_mul."""
    return layers * bsz * heads * dim * len_keys * o_mul


def score_bytes(seq_lens, G: int, D: int, e: int = 2) -> int:
    return sum(int(s) * G * D * e for s in seq_lens)


def attn_bytes(seq_lens, L: int, G: int, D: int, k: int, e: int = 2) -> int:
    return sum(L * G * min(k, int(s)) * D * e * 2 for s in seq_lens)


def step_bytes(seq_lens, L: int, G: int, D: int, k: int, e: int = 2) -> int:
    return score_bytes(seq_lens, G, D, e) + attn_bytes(seq_lens, L, G, D, k, e)


def step_flops(seq_lens, L: int, Hq: int, D: int, k: int) -> int:
    """2 flops per FMA: scoring Hq*D*S FMAs (Eq.3 with layers = 1), attention 2*L*Hq*k*D FMAs."""
    return sum(2 * Hq * D * int(s) + 4 * L * Hq * min(k, int(s)) * D for s in seq_lens)
