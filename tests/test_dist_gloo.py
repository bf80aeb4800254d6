"""World-size-2/3 gloo tests of the context-sharded step (O13) on CPU.

Each rank holds the strided shard t ≡ r (mod P) of the retrieval keys and of every KV
layer; the step's collectives (all-reduce MAX / SUM, all-gather of candidates and of
attention partials) run over torch.distributed/gloo with the oracle-backed CPU ops.  The
union of the ranks' selections must equal the single-device selection bit for bit and the
merged attention must equal single-device attention (fp64, 1e-9).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def global_inputs(S, seed):
    from paper_2512_00722_b200 import synth
    B, G, Hq, D, L = 1, 2, 8, 64, 2
    kr = synth.retrieval_keys(B, G, S, D, seed=seed)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=seed)
    qr = synth.retrieval_queries(1, B, Hq, G, D, seed=seed)[0]
    ql = synth.llm_queries(1, L, B, Hq, D, seed=seed)[0]
    return kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], qr, ql


def worker(rank, P, port, S, k, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ops import OracleOps
    from paper_2512_00722_b200 import dist as sdist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=P)
    kr, kl, vl, qr, ql = global_inputs(S, seed=3)
    st = sdist.make_shard(rank, P, kr, kl, vl, qr, ql, [S], k)
    pos, cnt, out, lse = sdist.run_distributed(OracleOps(), st)
    gids = [int(x) * P + rank for x in pos[0, 0, :int(cnt[0, 0])]] + \
           [int(x) * P + rank for x in pos[0, 1, :int(cnt[0, 1])]]
    allg = [None] * P
    dist.all_gather_object(allg, (pos.numpy(), cnt.numpy()))
    if rank == 0:
        np.savez(out_path, out=out.numpy(), lse=lse.numpy(),
                 pos=np.stack([a[0] for a in allg]), cnt=np.stack([a[1] for a in allg]))
    dist.barrier()
    dist.destroy_process_group()
    del gids


@pytest.mark.parametrize("P,S,k", [(2, 777, 96), (3, 1000, 128)])
def test_sharded_step_gloo(tmp_path, oracle, P, S, k):
    from paper_2512_00722_b200 import synth
    out_path = str(tmp_path / "res.npz")
    mp.start_processes(worker, args=(P, free_port(), S, k, out_path), nprocs=P, join=True,
                       start_method="spawn")
    res = np.load(out_path)
    kr, kl, vl, qr, ql = global_inputs(S, seed=3)
    scale = float(np.float32(1 / np.sqrt(64)))
    _, _, _, gs = oracle.score(synth.bf16_bits(qr), synth.bf16_bits(kr), [S], 2, scale)
    idx, _, cnt, _ = oracle.topk(gs, [S], k, force_last=True)
    for g in range(2):
        union = sorted(int(x) * P + r for r in range(P)
                       for x in res["pos"][r, 0, g, :res["cnt"][r, 0, g]])
        assert union == idx[0, g, :cnt[0, g]].tolist(), g
    oo, ol = oracle.sparse_attn(synth.bf16_bits(ql), [synth.bf16_bits(t) for t in kl],
                                [synth.bf16_bits(t) for t in vl], idx, cnt, scale)
    assert np.abs(res["out"] - oo).max() < 1e-9
    assert np.abs(res["lse"] - ol).max() < 1e-9


def test_shard_plan():
    from paper_2512_00722_b200 import dist as sdist
    for S in (1, 7, 1000, 1048576):
        for P in (1, 2, 3, 8):
            assert sum(sdist.local_len(S, P, r) for r in range(P)) == S
            last = S - 1
            r = sdist.owner(last, P)
            assert (last - r) // P == sdist.local_len(S, P, r) - 1  # last local position


def count_worker(rank, P, port, S, k, out_path):
    """One sharded step with every torch.distributed collective counted."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ops import OracleOps
    from paper_2512_00722_b200 import dist as sdist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=P)
    calls = []
    names = ("all_reduce", "all_gather", "all_gather_into_tensor", "broadcast", "reduce_scatter",
             "all_to_all", "all_gather_object", "reduce", "gather", "scatter")
    saved = {n: getattr(dist, n) for n in names if hasattr(dist, n)}

    def wrap(n, f):
        def g(*a, **kw):
            calls.append(n)
            return f(*a, **kw)
        return g
    for n, f in saved.items():
        setattr(dist, n, wrap(n, f))
    kr, kl, vl, qr, ql = global_inputs(S, seed=4)
    st = sdist.make_shard(rank, P, kr, kl, vl, qr, ql, [S], k)
    sdist.run_distributed(OracleOps(), st)
    for n, f in saved.items():
        setattr(dist, n, f)
    if rank == 0:
        with open(out_path, "w") as fh:
            fh.write(",".join(calls))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_uses_four_collectives(tmp_path):
    """the sharded step crosses the ranks four times -- all-reduce MAX,
    all-reduce SUM, one packed candidate all-gather, one packed (o, lse) all-gather."""
    out_path = str(tmp_path / "calls.txt")
    mp.start_processes(count_worker, args=(2, free_port(), 500, 64, out_path), nprocs=2, join=True,
                       start_method="spawn")
    calls = open(out_path).read().split(",")
    assert calls == ["all_reduce", "all_reduce", "all_gather_into_tensor", "all_gather_into_tensor"]
