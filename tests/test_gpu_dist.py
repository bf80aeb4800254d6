"""Context-sharded step (O13) through libspc with P ranks emulated on one GPU: the union of
the ranks' selections equals the single-device oracle selection bit for bit, and the
LSE-merged attention matches the oracle within 2e-3 (bf16)."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import dist as sdist
from paper_2512_00722_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_emulated_sharded_step(oracle, P):
    dev = torch.device("cuda")
    B, G, Hq, D, S, L, k = 1, 8, 32, 128, 6000, 3, 512
    kr = synth.retrieval_keys(B, G, S, D, seed=P, device=dev)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=P, device=dev)
    qr = synth.retrieval_queries(1, B, Hq, G, D, seed=P, device=dev)[0]
    ql = synth.llm_queries(1, L, B, Hq, D, seed=P, device=dev)[0]
    kl, vl = [kc[l] for l in range(L)], [vc[l] for l in range(L)]
    states = [sdist.make_shard(r, P, kr, kl, vl, qr, ql, [S], k) for r in range(P)]
    sel, out, lse = sdist.run_emulated(sdist.SpcOps(), states)
    torch.cuda.synchronize()
    scale = states[0].scale
    _, _, _, gs = oracle.score(synth.bf16_bits(qr), synth.bf16_bits(kr), [S], G, scale)
    idx, _, cnt, _ = oracle.topk(gs, [S], k, force_last=True)
    for g in range(G):
        union = sorted(int(x) * P + r for r in range(P)
                       for x in sel[r][0][0, g, :int(sel[r][1][0, g])].tolist())
        assert union == idx[0, g, :cnt[0, g]].tolist(), g
    oo, ol = oracle.sparse_attn(synth.bf16_bits(ql), [synth.bf16_bits(t) for t in kl],
                                [synth.bf16_bits(t) for t in vl], idx, cnt, scale)
    assert np.abs(out.cpu().numpy() - oo).max() <= 2e-3
    assert np.abs(lse.cpu().numpy() - ol).max() <= 1e-3


def _gloo_gpu_worker(rank, P, port, out_path):
    """One rank of a real multi-process sharded step on one GPU: libspc kernels (SpcOps) on
    cuda:0, the four collectives over gloo (NCCL needs one GPU per rank)."""
    import os
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2512_00722_b200 import dist as sd
    from paper_2512_00722_b200 import synth as sy
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=P)
    dev = torch.device("cuda", 0)
    B, G, Hq, D, S, L, k = 1, 8, 32, 128, 6000, 2, 512
    kr = sy.retrieval_keys(B, G, S, D, seed=11, device=dev)
    kc, vc = sy.llm_kv(L, B, G, S, D, seed=11, device=dev)
    qr = sy.retrieval_queries(1, B, Hq, G, D, seed=11, device=dev)[0]
    ql = sy.llm_queries(1, L, B, Hq, D, seed=11, device=dev)[0]
    st = sd.make_shard(rank, P, kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], qr, ql,
                       [S], k)
    pos, cnt, out, lse = sd.run_distributed(sd.SpcOps(), st)
    torch.cuda.synchronize()
    allg = [None] * P
    dist.all_gather_object(allg, (pos.cpu().numpy(), cnt.cpu().numpy()))
    if rank == 0:  # the global inputs too: the oracle must see the GPU-generated values
        np.savez(out_path, out=out.cpu().numpy(), lse=lse.cpu().numpy(),
                 pos=np.stack([a[0] for a in allg]), cnt=np.stack([a[1] for a in allg]),
                 kr=sy.bf16_bits(kr), kc=sy.bf16_bits(kc), vc=sy.bf16_bits(vc),
                 qr=sy.bf16_bits(qr), ql=sy.bf16_bits(ql))
    dist.barrier()
    dist.destroy_process_group()


def test_run_distributed_two_processes_one_gpu(oracle, tmp_path):
    """run_distributed (the four-collective step) with real libspc kernels in two processes:
    the union of the ranks' selections equals the oracle's, the merged attention within 2e-3."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    P, out_path = 2, str(tmp_path / "res.npz")
    mp.start_processes(_gloo_gpu_worker, args=(P, port, out_path), nprocs=P, join=True,
                       start_method="spawn")
    res = np.load(out_path)
    B, G, Hq, D, S, L, k = 1, 8, 32, 128, 6000, 2, 512
    kc, vc = res["kc"], res["vc"]
    scale = float(np.float32(1 / np.sqrt(D)))
    _, _, _, gs = oracle.score(res["qr"], res["kr"], [S], G, scale)
    idx, _, cnt, _ = oracle.topk(gs, [S], k, force_last=True)
    for g in range(G):
        union = sorted(int(x) * P + r for r in range(P)
                       for x in res["pos"][r, 0, g, :res["cnt"][r, 0, g]])
        assert union == idx[0, g, :cnt[0, g]].tolist(), g
    oo, ol = oracle.sparse_attn(res["ql"], [kc[l] for l in range(L)], [vc[l] for l in range(L)],
                                idx, cnt, scale)
    assert np.abs(res["out"] - oo).max() <= 2e-3
    assert np.abs(res["lse"] - ol).max() <= 1e-3
