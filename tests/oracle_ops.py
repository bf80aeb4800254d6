"""CPU backend for paper_2512_00722_b200.dist built on the oracle — TEST INFRASTRUCTURE.

Lets the sharded orchestration (collective points, id mapping, threshold merge, LSE merge)
run over torch.distributed/gloo on CPU, where libspc cannot run.  Each phase calls the
oracle on this rank's local shard; tensors are CPU torch tensors.
"""
import numpy as np
import torch

import oracle
from paper_2512_00722_b200 import synth


class OracleOps:
    def logits(self, st):
        lg, hm = oracle.logits(synth.bf16_bits(st.q_ret), synth.bf16_bits(st.kr), st.local_seq(),
                               st.G, st.scale)
        st.bufs["lg"] = lg
        return torch.from_numpy(hm.copy())

    def norm(self, st, head_max):
        F = oracle.norm(st.bufs["lg"], head_max.numpy(), st.local_seq())
        return torch.from_numpy(F)

    def group(self, st, head_max, sumfix):
        gs = oracle.group(st.bufs["lg"], head_max.numpy(), sumfix.numpy(), st.local_seq(), st.G)
        return torch.from_numpy(gs)

    def topk_local(self, st, gs):
        B, G, _ = gs.shape
        k = st.k
        val = np.zeros((B, G, k), np.float32)
        pos = np.full((B, G, k), -1, np.int32)
        cnt = np.zeros((B, G), np.int32)
        loc = st.local_seq()
        for b in range(B):
            fp = loc[b] - 1 if st.owns_last(b) else -1
            for g in range(G):
                p, v, _ = oracle.topk_row(gs[b, g, :loc[b]].numpy(), k, fp, st.P, st.rank)
                pos[b, g, :len(p)] = p
                val[b, g, :len(p)] = v
                cnt[b, g] = len(p)
        return torch.from_numpy(val), torch.from_numpy(pos), torch.from_numpy(cnt)

    def merge(self, st, cv, cp, cc):
        P, B, G, k = cv.shape
        th = np.zeros(B * G, np.uint64)
        for b in range(B):
            for g in range(G):
                vals, ids = [], []
                for p in range(P):
                    n = int(cc[p, b, g])
                    vals += cv[p, b, g, :n].tolist()
                    ids += (cp[p, b, g, :n].numpy().astype(np.int64) * P + p).tolist()
                if len(vals) > k:
                    _, _, t = oracle.topk_row(np.array(vals, np.float32), k,
                                              cand_id=np.array(ids, np.int32))
                    th[b * G + g] = t
        return torch.from_numpy(th.view(np.int64))

    def filter(self, st, pos, val, cnt, thresh):
        B, G, k = pos.shape
        th = thresh.numpy().view(np.uint64)
        out = np.full((B, G, k), -1, np.int32)
        oc = np.zeros((B, G), np.int32)
        for b in range(B):
            for g in range(G):
                keep = [int(x) for x, v in zip(pos[b, g, :int(cnt[b, g])].tolist(),
                                               val[b, g, :int(cnt[b, g])].tolist())
                        if oracle.composite(v, x * st.P + st.rank) >= th[b * G + g]]
                out[b, g, :len(keep)] = keep
                oc[b, g] = len(keep)
        return torch.from_numpy(out), torch.from_numpy(oc)

    def attn(self, st, pos, cnt):
        L = st.L
        o, lse = oracle.sparse_attn(synth.bf16_bits(st.q_llm),
                                    [synth.bf16_bits(t) for t in st.k_layers],
                                    [synth.bf16_bits(t) for t in st.v_layers],
                                    pos.numpy(), cnt.numpy(), st.scale, layers=range(L))
        return torch.from_numpy(o), torch.from_numpy(lse)

    def attn_merge(self, st, o_all, lse_all):
        P = o_all.shape[0]
        D = o_all.shape[-1]
        n = o_all[0].numel() // D
        out, lse = oracle.attn_merge(o_all.reshape(P, n, D).numpy(), lse_all.reshape(P, n).numpy())
        return (torch.from_numpy(out).view(o_all.shape[1:]),
                torch.from_numpy(lse).view(lse_all.shape[1:]))
