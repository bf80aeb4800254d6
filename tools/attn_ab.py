"""A/B of the two bf16 attention kernels on the config-B shape (tools only):
spc_sparse_decode_attn (pointer tables, per-warp cp.async rings) vs spc_sparse_decode_attn_kv
(TMA tile::gather4 producer + MMA consumer).  Three address-distinct KV copies rotated
launch to launch (each launch reads 256 MiB of selected rows from a 4 GiB cache).
Usage: python tools/attn_ab.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

_lib_arg = [a for a in sys.argv if a.startswith("--lib=")]
if _lib_arg:  # a debug build of libspc (tools/ only)
    spc._lib = spc.load_library(_lib_arg[0][6:])
    sys.argv.remove(_lib_arg[0])

dev = torch.device("cuda")
L, B, G, Hq, D, S, k = 32, 1, 8, 32, 128, 32768, 2048
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
NC = 3
copies = []
for c in range(NC):
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=10 + c, device=dev)
    copies.append((kc, vc, spc.ptr_table([kc[l] for l in range(L)], dev),
                   spc.ptr_table([vc[l] for l in range(L)], dev),
                   spc.KvDesc([kc[l] for l in range(L)], [vc[l] for l in range(L)])))
q = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
g = torch.Generator(device=dev).manual_seed(0)
idx = torch.sort(torch.rand(B, G, S, device=dev, generator=g).argsort(-1)[..., :k].to(torch.int32),
                 -1).values.contiguous()
cnt = torch.full((B, G), k, dtype=torch.int32, device=dev)
outs = {n: torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev) for n in ("ptr", "tma")}
lses = {n: torch.zeros((L, B, Hq), dtype=torch.float32, device=dev) for n in ("ptr", "tma")}
ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
nbytes = L * B * G * k * D * 2 * 2


LE = L


def launch(name, c):
    kc, vc, kt, vt, desc = copies[c % NC]
    if name == "ptr":
        spc.sparse_decode_attn(q, kt, vt, spc.KV_INDEXED, idx, cnt, S, k, 0.088, outs[name],
                               lses[name], ws, G, layer_end=LE)
    else:
        spc.sparse_decode_attn_kv(desc, q, spc.KV_INDEXED, idx, cnt, k, 0.088, outs[name],
                                  lses[name], ws, layer_end=LE)


for name in ("ptr", "tma"):
    launch(name, 0)
torch.cuda.synchronize()
print("max |tma - ptr| out %.3e  lse %.3e" % ((outs["tma"] - outs["ptr"]).abs().max().item(),
                                              (lses["tma"] - lses["ptr"]).abs().max().item()))
for rnd, LE in ((0, L), (1, L), (2, L // 2), (3, L // 4)):
    nbytes = LE * B * G * k * D * 2 * 2
    for name in ("ptr", "tma"):
        for c in range(6):
            launch(name, c)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for c in range(reps):
            launch(name, c)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        print(f"round {rnd} layers {LE} {name}: {us:7.2f} us per launch, {nbytes / us / 1e3:7.1f} GB/s")
