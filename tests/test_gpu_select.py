"""GPU parity of spc_topk / spc_topk_merge / spc_topk_filter (O7, O13), spc_elastic_diff (O8)
and spc_gather_kv (O9) against the CPU oracle: bit-exact indices, counts, thresholds,
diffs, slot maps and gathered bytes."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import spc, synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def gpu_topk(gs, seq, k, force=False, stride=1, offset=0):
    B, G, n = gs.shape
    gs_d = torch.as_tensor(gs).to(DEV)
    seq_d = torch.tensor(seq, dtype=torch.int32, device=DEV)
    idx = torch.zeros((B, G, k), dtype=torch.int32, device=DEV)
    val = torch.zeros((B, G, k), dtype=torch.float32, device=DEV)
    cnt = torch.zeros((B, G), dtype=torch.int32, device=DEV)
    th = torch.zeros((B, G), dtype=torch.int64, device=DEV)
    ws = spc.alloc_workspace(spc.topk_workspace(B, G, n, k), DEV)
    spc.topk(gs_d, seq_d, k, idx, cnt, ws, out_val=val, out_thresh=th, force_last=force,
             id_stride=stride, id_offset=offset)
    torch.cuda.synchronize()
    return (idx.cpu().numpy(), val.cpu().numpy(), cnt.cpu().numpy(),
            th.cpu().numpy().view(np.uint64))


def check_topk(oracle, gs, seq, k, force=False, stride=1, offset=0):
    idx, val, cnt, th = gpu_topk(gs, seq, k, force, stride, offset)
    oidx, oval, ocnt, oth = oracle.topk(gs, seq, k, force, stride, offset)
    assert np.array_equal(cnt, ocnt)
    assert np.array_equal(idx, oidx)
    assert np.array_equal(val.view(np.uint32), oval.view(np.uint32))
    B, G, n = gs.shape
    for b in range(B):
        for g in range(G):
            ln = min(seq[b], n)
            want = oth[b, g] if ln > k else 0  # 0 = no cut (everything kept)
            assert th[b, g] == want


def test_topk_random_rows_with_ties(oracle):
    rng = np.random.default_rng(0)
    for trial in range(12):
        B, G = 2, 3
        n = int(rng.integers(300, 20000))
        k = int(rng.integers(1, 2500))
        gs = rng.random((B, G, n)).astype(np.float32)
        if trial % 3 == 0:
            gs = (np.round(gs * 16) / 16).astype(np.float32)  # massive exact ties
        if trial % 4 == 1:
            gs = (gs ** 8).astype(np.float32)  # wide dynamic range
        seq = [n, int(rng.integers(1, n + 1))]
        check_topk(oracle, gs, seq, k, force=bool(trial % 2), stride=1 + trial % 3,
                   offset=trial % 2)


def test_topk_degenerate_all_equal_and_small(oracle):
    gs = np.full((1, 2, 30000), 0.25, np.float32)  # every element in one bin: row-scan fallback
    check_topk(oracle, gs, [30000], 2048)
    check_topk(oracle, gs, [30000], 2048, force=True)
    gs = np.random.default_rng(1).random((1, 1, 5)).astype(np.float32)
    check_topk(oracle, gs, [5], 8)   # k > S: everything
    check_topk(oracle, gs, [5], 5)   # k == S
    check_topk(oracle, gs, [1], 4, force=True)
    z = np.zeros((1, 1, 4096), np.float32)
    z[0, 0, ::7] = 1e-30
    check_topk(oracle, z, [4096], 1000)  # zeros and tiny values


def test_topk_on_real_scores_config_b(oracle):
    """The actual group scores of config B (S = 32768, G = 8, k = 2048)."""
    c = synth.CONFIGS["B"]
    kr = synth.retrieval_keys(1, c["G"], c["S"], c["D"], seed=7, device=DEV)
    q = synth.retrieval_queries(1, 1, c["Hq"], c["G"], c["D"], seed=7, device=DEV)[0]
    gs = torch.zeros((1, c["G"], c["S"]), dtype=torch.float32, device=DEV)
    lg = torch.zeros((1, c["Hq"], c["S"]), dtype=torch.float32, device=DEV)
    hm = torch.zeros((1, c["Hq"]), dtype=torch.float32, device=DEV)
    F = torch.zeros((1, c["Hq"]), dtype=torch.int64, device=DEV)
    seq = torch.tensor([c["S"]], dtype=torch.int32, device=DEV)
    ws = spc.alloc_workspace(spc.score_workspace(1, c["Hq"], c["S"]), DEV)
    spc.score(q, kr, seq, c["G"], 0.08838834764831845, lg, hm, F, gs, ws)
    check_topk(oracle, gs.cpu().numpy(), [c["S"]], c["k"], force=True)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_merge_and_filter_equal_global(oracle, P):
    """O13 on one GPU (emulated ranks): local top-k per strided shard with global ids, merged
    threshold, filtered lists; their union equals the single-device selection bit-exactly."""
    rng = np.random.default_rng(P)
    B, G, S, k = 1, 4, 6000, 512
    gs = (np.round(rng.random((B, G, S)) * 64) / 64).astype(np.float32)
    want, _, _, _ = oracle.topk(gs, [S], k, force_last=True)
    cv = np.zeros((P, B * G, k), np.float32)
    cp = np.zeros((P, B * G, k), np.int32)
    cc = np.zeros((P, B * G), np.int32)
    for r in range(P):
        loc = np.ascontiguousarray(gs[:, :, r::P])
        n_loc = loc.shape[2]
        owner_last = (S - 1) % P == r
        idx, val, cnt, _ = gpu_topk(loc, [n_loc], k, force=owner_last, stride=P, offset=r)
        cv[r], cp[r], cc[r] = val.reshape(B * G, k), idx.reshape(B * G, k), cnt.reshape(B * G)
    th = torch.zeros(B * G, dtype=torch.int64, device=DEV)
    spc.topk_merge(torch.from_numpy(cv).to(DEV), torch.from_numpy(cp).to(DEV),
                   torch.from_numpy(cc).to(DEV), k, th)
    union = [[] for _ in range(B * G)]
    for r in range(P):
        idx = torch.from_numpy(cp[r]).to(DEV)
        cnt = torch.from_numpy(cc[r]).to(DEV)
        spc.topk_filter(idx, torch.from_numpy(cv[r]).to(DEV), cnt, th, k, P, r)
        torch.cuda.synchronize()
        ii, nn = idx.cpu().numpy(), cnt.cpu().numpy()
        for row in range(B * G):
            union[row] += [int(x) * P + r for x in ii[row, :nn[row]]]
            assert np.all(np.diff(ii[row, :nn[row]]) > 0)  # stays ascending
    for row in range(B * G):
        assert sorted(union[row]) == want.reshape(B * G, k)[row].tolist()


def test_elastic_diff_random_walk(oracle):
    """Bit-exact load/evict lists and slot maps over a multi-step walk, INDEXED and SLOTS."""
    rng = np.random.default_rng(3)
    B, G, k, S = 2, 3, 300, 2000
    R = B * G
    prev = [np.zeros(0, np.int32) for _ in range(R)]
    slots_o = [np.full(k, -1, np.int32) for _ in range(R)]
    slot_tok = torch.full((B, G, k), -1, dtype=torch.int32, device=DEV)
    prev_d = torch.full((B, G, k), -1, dtype=torch.int32, device=DEV)
    prevc_d = torch.zeros((B, G), dtype=torch.int32, device=DEV)
    for step in range(25):
        cur = []
        for r in range(R):
            keep = prev[r][rng.random(len(prev[r])) < 0.8]
            n = min(k, len(keep) + int(rng.integers(0, 120))) if step % 5 else int(rng.integers(0, k))
            n = max(n, len(keep)) if step % 5 else n
            pool = np.setdiff1d(np.arange(S), keep)
            add = rng.choice(pool, size=max(0, n - len(keep)), replace=False)
            cur.append(np.sort(np.concatenate([keep, add]))[:n].astype(np.int32))
        cur_np = np.full((R, k), -1, np.int32)
        for r in range(R):
            cur_np[r, :len(cur[r])] = cur[r]
        cur_d = torch.from_numpy(cur_np.reshape(B, G, k)).to(DEV)
        curc_d = torch.tensor([len(c) for c in cur], dtype=torch.int32, device=DEV).view(B, G)
        lt = torch.zeros((B, G, k), dtype=torch.int32, device=DEV)
        ls = torch.zeros((B, G, k), dtype=torch.int32, device=DEV)
        et = torch.zeros((B, G, k), dtype=torch.int32, device=DEV)
        nl = torch.zeros((B, G), dtype=torch.int32, device=DEV)
        ne = torch.zeros((B, G), dtype=torch.int32, device=DEV)
        spc.elastic_diff(prev_d, prevc_d, cur_d, curc_d, lt, nl, slot_tok=slot_tok, load_slot=ls,
                         evict_tok=et, n_evict=ne)
        torch.cuda.synchronize()
        lt_, ls_, et_ = (x.cpu().numpy().reshape(R, k) for x in (lt, ls, et))
        nl_, ne_ = nl.cpu().numpy().reshape(R), ne.cpu().numpy().reshape(R)
        st_ = slot_tok.cpu().numpy().reshape(R, k)
        for r in range(R):
            o = oracle.elastic_diff_row(prev[r], cur[r], k, slots_o[r])
            assert o["status"] == 0
            assert nl_[r] == o["n_load"] and ne_[r] == o["n_evict"]
            assert np.array_equal(lt_[r], o["load_tok"])
            assert np.array_equal(et_[r], o["evict_tok"])
            assert np.array_equal(ls_[r], o["load_slot"])
            assert np.array_equal(st_[r], o["slot_tok"])
            slots_o[r] = o["slot_tok"]
            kept = set(prev[r]) & set(cur[r])
            assert sorted(kept | set(lt_[r, :nl_[r]].tolist())) == cur[r].tolist()  # union inv.
        prev = cur
        prev_d, prevc_d = cur_d, curc_d


def test_gather_kv_bytes_exact(oracle):
    """O9: slot rows equal the source rows byte for byte, every layer; the source may be pinned
    host memory (zero-copy)."""
    L, B, G, D, Smax, k = 3, 2, 2, 128, 500, 64
    for host in (False, True):
        kc, vc = synth.llm_kv(L, B, G, Smax, D, seed=9)
        if host:
            kc, vc = kc.pin_memory(), vc.pin_memory()
        else:
            kc, vc = kc.to(DEV), vc.to(DEV)
        kb = torch.zeros((L, B, G, k, D), dtype=torch.bfloat16, device=DEV)
        vb = torch.zeros_like(kb)
        rng = np.random.default_rng(4)
        lt = np.full((B * G, k), -1, np.int32)
        ls = np.full((B * G, k), -1, np.int32)
        nl = np.zeros(B * G, np.int32)
        for r in range(B * G):
            n = int(rng.integers(0, k + 1))
            lt[r, :n] = np.sort(rng.choice(Smax, n, replace=False))
            ls[r, :n] = rng.permutation(k)[:n]
            nl[r] = n
        spc.gather_kv(spc.ptr_table([kc[l] for l in range(L)], DEV),
                      spc.ptr_table([vc[l] for l in range(L)], DEV), L, B, G, D, Smax, k,
                      torch.from_numpy(lt).to(DEV), torch.from_numpy(ls).to(DEV),
                      torch.from_numpy(nl).to(DEV), spc.ptr_table([kb[l] for l in range(L)], DEV),
                      spc.ptr_table([vb[l] for l in range(L)], DEV))
        torch.cuda.synchronize()
        kcc, vcc, kbc, vbc = kc.cpu(), vc.cpu(), kb.cpu(), vb.cpu()
        for l in range(L):
            for r in range(B * G):
                b, g = divmod(r, G)
                for i in range(nl[r]):
                    assert torch.equal(kbc[l, b, g, ls[r, i]], kcc[l, b, g, lt[r, i]])
                    assert torch.equal(vbc[l, b, g, ls[r, i]], vcc[l, b, g, lt[r, i]])


@pytest.mark.parametrize("D", [128, 64])
def test_gather_kv_strided_token_major_bytes_exact(D):
    """O9 from a TOKEN-MAJOR source (one record [L][2][D] per token, the offloaded-KV layout
    of config D): spc_gather_kv_strided copies the K and V rows of every layer in range
    byte for byte, from device or pinned host memory, for empty, partial and full loads."""
    L, B, G, Smax, k = 5, 2, 3, 300, 96
    rec = synth.normal_bf16((B, G, Smax, L, 2, D), 31)
    for host in (False, True):
        src = rec.pin_memory() if host else rec.to(DEV)
        base, esz = src.data_ptr(), 2
        k_tab = torch.tensor([base + l * 2 * D * esz for l in range(L)], dtype=torch.int64,
                             device=DEV)
        v_tab = k_tab + D * esz
        kb = torch.zeros((L, B, G, k, D), dtype=torch.bfloat16, device=DEV) - 1
        vb = torch.zeros_like(kb) - 1
        rng = np.random.default_rng(5)
        lt = np.full((B * G, k), -1, np.int32)
        ls = np.full((B * G, k), -1, np.int32)
        nl = np.array([0, k, 1, 37, 64, 95][:B * G], np.int32)
        for r in range(B * G):
            n = int(nl[r])
            lt[r, :n] = np.sort(rng.choice(Smax, n, replace=False))
            ls[r, :n] = rng.permutation(k)[:n]
        l0, l1 = (0, L) if host else (1, 4)
        spc.gather_kv_strided(k_tab, v_tab, L * 2 * D, Smax * L * 2 * D, L, B, G, D, k,
                              torch.from_numpy(lt).to(DEV), torch.from_numpy(ls).to(DEV),
                              torch.from_numpy(nl).to(DEV), spc.ptr_table([kb[l] for l in range(L)], DEV),
                              spc.ptr_table([vb[l] for l in range(L)], DEV), layer_begin=l0,
                              layer_end=l1)
        torch.cuda.synchronize()
        kbc, vbc = kb.cpu(), vb.cpu()
        expect_k = torch.zeros_like(kbc) - 1
        expect_v = torch.zeros_like(vbc) - 1
        for l in range(l0, l1):
            for r in range(B * G):
                b, g = divmod(r, G)
                n = int(nl[r])
                expect_k[l, b, g, ls[r, :n]] = rec[b, g, lt[r, :n], l, 0]
                expect_v[l, b, g, ls[r, :n]] = rec[b, g, lt[r, :n], l, 1]
        assert torch.equal(kbc.view(torch.int16), expect_k.view(torch.int16))
        assert torch.equal(vbc.view(torch.int16), expect_v.view(torch.int16))


@pytest.mark.parametrize("alpha,G,S,k", [(4, 8, 32768, 2048), (2, 3, 5000, 700), (8, 1, 300, 512),
                                         (1, 4, 20000, 64)])
def test_fused_select_equals_separate_calls(oracle, alpha, G, S, k):
    """spc_select (one launch) is bit-identical to spc_score(NORM|GROUP) + spc_topk +
    spc_elastic_diff, and to the oracle, over two consecutive steps."""
    B, D = 2, 128
    Hq = alpha * G
    kr = synth.retrieval_keys(B, G, S, D, seed=alpha + S, device=DEV)
    qs = synth.retrieval_queries(2, B, Hq, G, D, seed=alpha + S, device=DEV)
    seq = torch.tensor([S, max(1, S // 3)], dtype=torch.int32, device=DEV)
    f32, i32 = torch.float32, torch.int32
    mk = lambda *s, dt=f32: torch.zeros(s, dtype=dt, device=DEV)
    ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), DEV)
    wt = spc.alloc_workspace(spc.topk_workspace(B, G, S, k), DEV)
    prev_a, prevc_a = torch.full((B, G, k), -1, dtype=i32, device=DEV), mk(B, G, dt=i32)
    prev_b, prevc_b = prev_a.clone(), prevc_a.clone()
    for step in range(2):
        lg, hm = mk(B, Hq, S), mk(B, Hq)
        spc.score(qs[step], kr, seq, G, 0.088, lg, hm, mk(B, Hq, dt=torch.int64), mk(B, G, S), ws,
                  phases=spc.SCORE_LOGITS)
        # separate calls
        Fa, gsa = mk(B, Hq, dt=torch.int64), mk(B, G, S)
        spc.score(qs[step], kr, seq, G, 0.088, lg, hm, Fa, gsa, ws,
                  phases=spc.SCORE_NORM | spc.SCORE_GROUP)
        ia, ca = mk(B, G, k, dt=i32), mk(B, G, dt=i32)
        spc.topk(gsa, seq, k, ia, ca, wt, force_last=True)
        lta, nla, eta, nea = mk(B, G, k, dt=i32), mk(B, G, dt=i32), mk(B, G, k, dt=i32), mk(B, G, dt=i32)
        spc.elastic_diff(prev_a, prevc_a, ia, ca, lta, nla, evict_tok=eta, n_evict=nea)
        # fused
        Fb, gsb = mk(B, Hq, dt=torch.int64), mk(B, G, S) - 1
        ib, cb = mk(B, G, k, dt=i32), mk(B, G, dt=i32)
        ltb, nlb, etb, neb = mk(B, G, k, dt=i32), mk(B, G, dt=i32), mk(B, G, k, dt=i32), mk(B, G, dt=i32)
        spc.select(lg, hm, seq, G, k, Fb, gsb, ib, cb, prev_b, prevc_b, ltb, nlb, etb, neb,
                   force_last=True)
        torch.cuda.synchronize()
        for x, y in ((Fa, Fb), (ia, ib), (ca, cb), (lta, ltb), (nla, nlb), (eta, etb), (nea, neb)):
            assert torch.equal(x, y)
        assert torch.equal(gsa.view(torch.int32), gsb.view(torch.int32))
        oidx, _, ocnt, _ = oracle.topk(gsa.cpu().numpy(), seq.cpu().tolist(), k, force_last=True)
        assert np.array_equal(ib.cpu().numpy(), oidx)
        prev_a, prevc_a, prev_b, prevc_b = ia, ca, ib, cb


def _select_both(lg, hm, seq, G, k, prev=None, force=True):
    """Run the separate calls and spc_select on the same logits; assert bit-identity."""
    B, Hq, S = lg.shape
    f32, i32 = torch.float32, torch.int32
    mk = lambda *s, dt=f32: torch.zeros(s, dtype=dt, device=DEV)  # noqa: E731
    if prev is None:
        prev = (torch.full((B, G, k), -1, dtype=i32, device=DEV), mk(B, G, dt=i32))
    ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), DEV)
    wt = spc.alloc_workspace(spc.topk_workspace(B, G, S, k), DEV)
    q = torch.zeros((B, Hq, 64), dtype=torch.bfloat16, device=DEV)
    kr = torch.zeros((B, G, S, 64), dtype=torch.bfloat16, device=DEV)
    Fa, gsa = mk(B, Hq, dt=torch.int64), mk(B, G, S)
    spc.score(q, kr, seq, G, 1.0, lg, hm, Fa, gsa, ws, phases=spc.SCORE_NORM | spc.SCORE_GROUP)
    ia, ca = mk(B, G, k, dt=i32), mk(B, G, dt=i32)
    spc.topk(gsa, seq, k, ia, ca, wt, force_last=force)
    outs_a = [mk(B, G, k, dt=i32), mk(B, G, dt=i32), mk(B, G, k, dt=i32), mk(B, G, dt=i32)]
    spc.elastic_diff(prev[0], prev[1], ia, ca, outs_a[0], outs_a[1], evict_tok=outs_a[2],
                     n_evict=outs_a[3])
    Fb, gsb = mk(B, Hq, dt=torch.int64) - 7, mk(B, G, S) - 1
    ib, cb = mk(B, G, k, dt=i32) - 5, mk(B, G, dt=i32)
    outs_b = [mk(B, G, k, dt=i32) - 3, mk(B, G, dt=i32), mk(B, G, k, dt=i32) - 3, mk(B, G, dt=i32)]
    spc.select(lg, hm, seq, G, k, Fb, gsb, ib, cb, prev[0], prev[1], outs_b[0], outs_b[1],
               outs_b[2], outs_b[3], force_last=force)
    torch.cuda.synchronize()
    assert torch.equal(Fa, Fb)
    assert torch.equal(gsa.view(torch.int32), gsb.view(torch.int32))
    assert torch.equal(ia, ib) and torch.equal(ca, cb)
    for x, y in zip(outs_a, outs_b):
        assert torch.equal(x, y)
    return gsa, ia, ca


def _logits_case(kind, B, Hq, S, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    if kind == "flat":            # every score equal: clamped top bin, ties broken by id bits
        lg = torch.zeros((B, Hq, S))
    elif kind == "two_level":     # a few spikes over a flat floor: tiny threshold buckets
        lg = torch.zeros((B, Hq, S))
        lg[:, :, torch.randperm(S, generator=g)[:S // 50]] = 3.0
    elif kind == "quantised":     # 17 distinct logits: large exact-tie buckets
        lg = torch.randint(0, 17, (B, Hq, S), generator=g).float() * 0.25
    elif kind == "wide":          # scores spanning > 32 binades below the max (bottom clamp)
        lg = -torch.rand((B, Hq, S), generator=g) * 80.0
        lg[:, :, 0] = 0.0
    else:                         # smooth random
        lg = torch.randn((B, Hq, S), generator=g) * 2.0
    return lg.to(DEV)


@pytest.mark.parametrize("kind", ["flat", "two_level", "quantised", "wide", "randn"])
@pytest.mark.parametrize("alpha,G,S,k,lens", [(4, 2, 8192, 1024, [8192, 3001]),
                                              (2, 1, 1000, 1000, [999]),
                                              (1, 3, 40000, 2048, [40000, 1]),
                                              (8, 1, 4096, 300, [0])])
def test_fused_select_adversarial(oracle, kind, alpha, G, S, k, lens):
    B, Hq = len(lens), alpha * G
    lg = _logits_case(kind, B, Hq, S, seed=S + alpha)
    seq = torch.tensor(lens, dtype=torch.int32, device=DEV)
    hm = torch.zeros((B, Hq), device=DEV)
    for b, n in enumerate(lens):
        if n > 0:
            hm[b] = lg[b, :, :n].max(-1).values
    gs, idx, cnt = _select_both(lg, hm, seq, G, k)
    oidx, _, ocnt, _ = oracle.topk(gs.cpu().numpy(), lens, k, force_last=True)
    assert np.array_equal(idx.cpu().numpy(), oidx) and np.array_equal(cnt.cpu().numpy(), ocnt)
    # a second step against this selection (elastic diff with a non-empty previous list)
    lg2 = lg + 0.01 * _logits_case("randn", B, Hq, S, seed=S + 1)
    hm2 = torch.zeros((B, Hq), device=DEV)
    for b, n in enumerate(lens):
        if n > 0:
            hm2[b] = lg2[b, :, :n].max(-1).values
    _select_both(lg2, hm2, seq, G, k, prev=(idx, cnt))


def test_fused_select_rejects_unsupported():
    B, G, Hq, k = 1, 1, 4, 64
    for S in (135172, 1001):  # beyond 8 * 16896 tokens; not a multiple of 4
        lg = torch.zeros((B, Hq, S), device=DEV)
        z = lambda *s, dt=torch.int32: torch.zeros(s, dtype=dt, device=DEV)  # noqa: E731
        with pytest.raises(spc.SpcError):
            spc.select(lg, z(B, Hq, dt=torch.float32), torch.tensor([S], dtype=torch.int32,
                       device=DEV), G, k, z(B, Hq, dt=torch.int64), z(B, G, S, dt=torch.float32),
                       z(B, G, k), z(B, G), z(B, G, k), z(B, G), z(B, G, k), z(B, G))


def test_maximum_sizes(oracle):
    """Upper limits of the ABI: k = SPC_MAX_K (4096) for the top-k, and the fused select at its
    largest supported row (Smax = 135168) with k = 4096 -- bit-identical to the oracle / the
    separate calls, with a ragged second request."""
    rng = np.random.default_rng(11)
    gs = rng.random((1, 2, 60000)).astype(np.float32) ** 4
    check_topk(oracle, gs, [60000], spc.MAX_K, force=True)
    # long rows, few of them: the 16-CTA cluster path (B*G*16 <= SMs, n >= 65536)
    gl = (rng.random((2, 3, 300000)).astype(np.float32) ** 6)
    gl[0, 1, 1000:1200] = gl[0, 1, 5]  # exact ties around the threshold
    check_topk(oracle, gl, [300000, 123457], 2048, force=True, stride=3, offset=1)
    B, G, Hq, S, k = 2, 1, 4, 135168, spc.MAX_K
    g = torch.Generator(device="cpu").manual_seed(3)
    lg = (torch.randn((B, Hq, S), generator=g) * 2).to(DEV)
    seq = torch.tensor([S, 70001], dtype=torch.int32, device=DEV)
    hm = torch.stack([lg[b, :, :int(seq[b])].amax(dim=1) for b in range(B)]).contiguous()
    gsa, ia, ca = _select_both(lg, hm, seq, G, k)
    oidx, _, ocnt, _ = oracle.topk(gsa.cpu().numpy(), seq.cpu().tolist(), k, force_last=True)
    assert np.array_equal(ia.cpu().numpy(), oidx) and np.array_equal(ca.cpu().numpy(), ocnt)
