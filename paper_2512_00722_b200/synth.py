"""Seeded synthetic workloads (shared by tests, bench and smoke).

This module holds NO arithmetic of the method: only random numbers and tensor
layout.  It is the one module both sides (the CUDA path and the CPU oracle)
may use; the oracle receives the exact bytes generated here.

Recipe, shaped like a long reasoning trace of
DeepSeek-R1-Distill-Llama-8B (GQA 32 q / 8 kv heads, d = 128):

* retrieval keys   Kr[b,g,t] = bf16(mu_g + z_t + beta * u_g * [t < N_SINK]),
  mu_g ~ N(0, 0.25 I) (a common per-group key bias), z_t ~ N(0, I),
  u_g a random unit vector per group, beta = 4 (attention sinks).
* retrieval queries: AR(1) drift a_s = rho a_{s-1} + sqrt(1-rho^2) xi_s with
  rho = 0.98 (adjacent decode steps look at nearly the same context),
  q_s[b,h] = bf16(Q_SCALE * (a_s[b,h] + 0.5 u_{g(h)})), Q_SCALE = 3.
* LLM K/V and LLM queries: bf16 N(0, 1).
* tie tests: duplicate key rows (``duplicate_rows``).
"""
from __future__ import annotations

import math

import torch

N_SINK = 4
SINK_BETA = 4.0
RHO = 0.98
Q_SCALE = 3.0
BASE_SEED = 20251201

# Workload shapes (BASELINE.json configs). L = LLM layers, G = KV groups,
# Hq = query heads, D = head dim, S = context, k = budget, B = batch.
CONFIGS = {
    "A": dict(name="tiny", B=1, L=1, Hq=4, G=1, D=64, S=4096, k=256),
    "B": dict(name="llama8b-32k", B=1, L=32, Hq=32, G=8, D=128, S=32768, k=2048),
    "C": dict(name="llama8b-128k-b16-growing", B=16, L=32, Hq=32, G=8, D=128, S=131072, k=2048),
    "D": dict(name="llama8b-256k-b32-offload", B=32, L=32, Hq=32, G=8, D=128, S=262144, k=2048),
    "E": dict(name="llama8b-1m-sharded", B=1, L=32, Hq=32, G=8, D=128, S=1048576, k=2048),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _randn(shape, gen, device, dtype=torch.float32):
    return torch.randn(shape, generator=gen, device=device, dtype=dtype)


def group_dirs(G: int, D: int, seed: int, device="cpu") -> torch.Tensor:
    """u_g: one random unit vector per KV group, [G][D] f32."""
    g = _gen(seed * 7 + 1, device)
    u = _randn((G, D), g, device)
    return u / u.norm(dim=-1, keepdim=True)


def retrieval_keys(B: int, G: int, Smax: int, D: int, seed: int, device="cpu",
                   chunk_rows: int = 1 << 22) -> torch.Tensor:
    """Kr [B][G][Smax][D] bf16 (see module docstring)."""
    u = group_dirs(G, D, seed, device)
    gm = _gen(seed * 7 + 2, device)
    mu = 0.5 * _randn((B, G, 1, D), gm, device)
    out = torch.empty((B, G, Smax, D), dtype=torch.bfloat16, device=device)
    gz = _gen(seed * 7 + 3, device)
    step = max(1, chunk_rows // max(1, B * G))
    for t0 in range(0, Smax, step):
        t1 = min(Smax, t0 + step)
        z = _randn((B, G, t1 - t0, D), gz, device)
        z += mu
        if t0 < N_SINK:
            z[:, :, : N_SINK - t0] += SINK_BETA * u[None, :, None, :]
        out[:, :, t0:t1] = z.to(torch.bfloat16)
    return out


def retrieval_queries(steps: int, B: int, Hq: int, G: int, D: int, seed: int,
                      device="cpu") -> torch.Tensor:
    """q [steps][B][Hq][D] bf16: AR(1) drifting queries (module docstring)."""
    u = group_dirs(G, D, seed, device)
    alpha = Hq // G
    ug = u.repeat_interleave(alpha, dim=0)  # [Hq][D]
    gq = _gen(seed * 7 + 4, device)
    a = _randn((B, Hq, D), gq, device)
    c = math.sqrt(1.0 - RHO * RHO)
    out = torch.empty((steps, B, Hq, D), dtype=torch.bfloat16, device=device)
    for s in range(steps):
        if s:
            a = RHO * a + c * _randn((B, Hq, D), gq, device)
        out[s] = (Q_SCALE * (a + 0.5 * ug[None])).to(torch.bfloat16)
    return out


def normal_bf16(shape, seed: int, device="cpu", dtype=torch.bfloat16,
                chunk: int = 1 << 26) -> torch.Tensor:
    """bf16 (or f32) N(0,1) tensor, generated in chunks (LLM K/V, LLM queries)."""
    g = _gen(seed, device)
    out = torch.empty(shape, dtype=dtype, device=device)
    flat = out.view(-1)
    n = flat.numel()
    for i in range(0, n, chunk):
        j = min(n, i + chunk)
        flat[i:j] = _randn((j - i,), g, device).to(dtype)
    return out


def llm_queries(steps: int, L: int, B: int, Hq: int, D: int, seed: int, device="cpu",
                dtype=torch.bfloat16) -> torch.Tensor:
    """q_llm [steps][L][B][Hq][D]."""
    return normal_bf16((steps, L, B, Hq, D), seed * 7 + 5, device, dtype)


def llm_kv(L: int, B: int, G: int, rows: int, D: int, seed: int, device="cpu",
           dtype=torch.bfloat16):
    """(K, V) each [L][B][G][rows][D]."""
    k = normal_bf16((L, B, G, rows, D), seed * 7 + 6, device, dtype)
    v = normal_bf16((L, B, G, rows, D), seed * 7 + 8, device, dtype)
    return k, v


def duplicate_rows(kr: torch.Tensor, n_dup: int, seed: int) -> torch.Tensor:
    """Copy n_dup random key rows over other rows of each (b,g) to create exact score ties."""
    B, G, S, D = kr.shape
    g = _gen(seed * 7 + 9, "cpu")
    out = kr.clone()
    for b in range(B):
        for gg in range(G):
            src = torch.randint(0, S, (n_dup,), generator=g)
            dst = torch.randint(0, S, (n_dup,), generator=g)
            out[b, gg, dst.to(kr.device)] = out[b, gg, src.to(kr.device)]
    return out


def bf16_bits(t: torch.Tensor):
    """Raw bf16 bit patterns as a numpy uint16 array on the host."""
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view("uint16")


def retrieval_head_weights(V: int, H: int, Hq: int, G: int, D: int, seed: int, device="cpu"):
    """Random-init weights of the retrieval head's front-end (NEXT-1; the trained EAGLE-3 DLM
    weights are out of scope): embedding [V][H] ~ N(0, 1), RMSNorm weight [H] ~
    1 + N(0, 0.05^2), W_qk [(Hq+G)*D][H] ~ N(0, 1/H) (unit-variance projections), all bf16."""
    emb = normal_bf16((V, H), seed * 11 + 1, device)
    norm_w = (1.0 + 0.05 * normal_bf16((H,), seed * 11 + 2, device, torch.float32)).to(torch.bfloat16)
    w_qk = (normal_bf16(((Hq + G) * D, H), seed * 11 + 3, device, torch.float32)
            * (1.0 / math.sqrt(H))).to(torch.bfloat16)
    return emb, norm_w, w_qk


def tokens(steps: int, B: int, V: int, seed: int, device="cpu") -> torch.Tensor:
    """Token ids [steps][B] int32, uniform over the vocabulary."""
    g = _gen(seed * 11 + 4, "cpu")
    return torch.randint(0, V, (steps, B), generator=g, dtype=torch.int32).to(device)


# LLM decoder shape for NEXT-4 (DeepSeek-R1-Distill-Llama-8B = Llama-3.1-8B architecture)
LLAMA8B = dict(L=32, H=4096, Hq=32, G=8, D=128, F=14336, V=128256, rope_base=500000.0, eps=1e-5)


def llm_weights(L: int, H: int, Hq: int, G: int, D: int, F: int, V: int, seed: int,
                device="cpu"):
    """Random-init weights of a Llama-style decoder (NEXT-4; trained weights are out of scope,
    DESIGN.md §5), nn.Linear layout [out][in], all bf16: emb [V][H] ~ N(0, 1); per layer
    ln1 / ln2 [H] ~ 1 + N(0, 0.05^2), w_qkv [(Hq + 2G) D][H], w_o [H][Hq D], w_gu [2F][H]
    (gate rows then up rows), w_down [H][F], each ~ N(0, 1/in); final norm [H]; lm_head [V][H]
    ~ N(0, 1/H)."""
    def lin(o, i, s):
        return normal_bf16((o, i), s, device).mul_(1.0 / math.sqrt(i))

    def norm(s):
        return (1.0 + 0.05 * normal_bf16((H,), s, device, torch.float32)).to(torch.bfloat16)

    base = seed * 13
    w = dict(emb=normal_bf16((V, H), base + 1, device), ln1=[], ln2=[], w_qkv=[], w_o=[],
             w_gu=[], w_down=[])
    for l in range(L):
        s = base + 100 * (l + 1)
        w["ln1"].append(norm(s + 1))
        w["ln2"].append(norm(s + 2))
        w["w_qkv"].append(lin((Hq + 2 * G) * D, H, s + 3))
        w["w_o"].append(lin(H, Hq * D, s + 4))
        w["w_gu"].append(lin(2 * F, H, s + 5))
        w["w_down"].append(lin(H, F, s + 6))
    w["norm"] = norm(base + 2)
    w["lm_head"] = lin(V, H, base + 3)
    return w
