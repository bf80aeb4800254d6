"""SPC_DEBUG device-side contract checks (include/spc.h "Errors"): libspc_debug.so records
the first violated data-dependent contract on the device and spc_check_device_errors()
returns it -- one test per error, plus a clean step that reports none."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import build, spc, synth
from paper_2512_00722_b200.pipeline import DecodeStep

pytestmark = pytest.mark.gpu
DEV = "cuda"
OK, E_BUDGET, E_RANGE, E_STATE = 0, 3, 4, 5
i32 = torch.int32


@pytest.fixture()
def dbg():
    keep = spc._lib
    spc._lib = spc.load_library(build.build_debug())
    assert spc.lib().spc_debug_build() == 1
    assert spc.check_device_errors() == OK  # nothing pending
    yield spc
    spc.check_device_errors()
    spc._lib = keep


def z(*s, dt=i32, fill=0):
    return torch.full(s, fill, dtype=dt, device=DEV)


def test_release_build_has_no_device_checks():
    assert spc.lib().spc_debug_build() == 0
    assert spc.check_device_errors() == OK


def test_clean_step_reports_nothing(dbg):
    c = synth.CONFIGS["A"]
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    kr = synth.retrieval_keys(B, G, S, D, seed=1, device=DEV)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=DEV)
    qr = synth.retrieval_queries(2, B, Hq, G, D, seed=1, device=DEV)
    ql = synth.llm_queries(1, L, B, Hq, D, seed=1, device=DEV)[0]
    st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)],
                    torch.full((B,), S, dtype=i32, device=DEV), L, Hq, k)
    for s in range(2):
        st.step(qr[s], ql)
    assert dbg.check_device_errors() == OK


def test_attention_index_out_of_range(dbg):
    """a selected index >= the cache rows is SPC_E_RANGE (both attention kernels)."""
    L, B, G, Hq, D, rows, k = 1, 1, 1, 4, 128, 1000, 64
    kc, vc = synth.llm_kv(L, B, G, rows, D, seed=2, device=DEV)
    q = synth.llm_queries(1, L, B, Hq, D, seed=2, device=DEV)[0]
    idx = torch.arange(k, dtype=i32, device=DEV).view(1, 1, k).clone()
    idx[0, 0, 10] = rows + 5
    cnt = z(1, 1, fill=k)
    out, lse = torch.zeros((L, B, Hq, D), device=DEV), torch.zeros((L, B, Hq), device=DEV)
    ws = dbg.alloc_workspace(dbg.attn_workspace(L, B, Hq, D, k), DEV)
    desc = dbg.KvDesc([kc[0]], [vc[0]])
    dbg.sparse_decode_attn_kv(desc, q, dbg.KV_INDEXED, idx, cnt, k, 0.1, out, lse, ws)
    assert dbg.check_device_errors() == E_RANGE
    dbg.sparse_decode_attn(q, dbg.ptr_table([kc[0]], DEV), dbg.ptr_table([vc[0]], DEV),
                           dbg.KV_INDEXED, idx, cnt, rows, k, 0.1, out, lse, ws, G)
    assert dbg.check_device_errors() == E_RANGE
    assert "attn" in dbg.lib().spc_last_cuda_error().decode()


def test_diff_unsorted_list(dbg):
    """index lists are ascending sets; an unsorted one is SPC_E_STATE."""
    k = 8
    prev = torch.tensor([[[1, 5, 3, 7, -1, -1, -1, -1]]], dtype=i32, device=DEV)
    cur = torch.tensor([[[1, 2, 3, 4, -1, -1, -1, -1]]], dtype=i32, device=DEV)
    lt, nl = z(1, 1, k), z(1, 1)
    dbg.elastic_diff(prev, z(1, 1, fill=4), cur, z(1, 1, fill=4), lt, nl)
    assert dbg.check_device_errors() == E_STATE


def test_diff_slot_map_inconsistent_with_previous_set(dbg):
    """the slot map must hold exactly the previous set; otherwise SPC_E_STATE."""
    k = 4
    prev = torch.tensor([[[2, 4, 6, -1]]], dtype=i32, device=DEV)
    cur = torch.tensor([[[2, 4, 8, -1]]], dtype=i32, device=DEV)
    slot = torch.tensor([[[2, 9, 6, -1]]], dtype=i32, device=DEV)  # 9 is not in prev
    lt, ls, nl = z(1, 1, k), z(1, 1, k), z(1, 1)
    dbg.elastic_diff(prev, z(1, 1, fill=3), cur, z(1, 1, fill=3), lt, nl, slot_tok=slot, load_slot=ls)
    assert dbg.check_device_errors() == E_STATE


def test_gather_index_out_of_range(dbg):
    """S:178 gather_kv: a load token beyond the source rows is SPC_E_RANGE (and not read)."""
    L, B, G, D, rows, k = 1, 1, 1, 128, 100, 8
    kc, vc = synth.llm_kv(L, B, G, rows, D, seed=3, device=DEV)
    kb, vb = torch.zeros((L, B, G, k, D), dtype=torch.bfloat16, device=DEV), \
        torch.zeros((L, B, G, k, D), dtype=torch.bfloat16, device=DEV)
    lt = torch.tensor([[[5, 150, -1, -1, -1, -1, -1, -1]]], dtype=i32, device=DEV)
    ls = torch.tensor([[[0, 1, -1, -1, -1, -1, -1, -1]]], dtype=i32, device=DEV)
    dbg.gather_kv(dbg.ptr_table([kc[0]], DEV), dbg.ptr_table([vc[0]], DEV), L, B, G, D, rows, k,
                  lt, ls, z(1, 1, fill=2), dbg.ptr_table([kb[0]], DEV), dbg.ptr_table([vb[0]], DEV))
    assert dbg.check_device_errors() == E_RANGE
    assert torch.equal(kb[0, 0, 0, 0], kc[0, 0, 0, 5])  # the valid row was copied


def test_select_unsorted_previous_selection(dbg):
    B, G, Hq, S, k = 1, 1, 4, 4096, 16
    lg = torch.randn((B, Hq, S), device=DEV)
    hm = lg.amax(-1)
    prev = torch.full((B, G, k), -1, dtype=i32, device=DEV)
    prev[0, 0, :3] = torch.tensor([30, 10, 20], dtype=i32)
    dbg.select(lg, hm, z(B, fill=S), G, k, z(B, Hq, dt=torch.int64), torch.zeros((B, G, S), device=DEV),
               z(B, G, k), z(B, G), prev, z(B, G, fill=3), z(B, G, k), z(B, G))
    assert dbg.check_device_errors() == E_STATE


def test_score_nan_key(dbg):
    """Reading R20: a NaN key makes a NaN logit: SPC_E_RANGE."""
    B, G, Hq, D, S = 1, 1, 4, 64, 512
    kr = synth.retrieval_keys(B, G, S, D, seed=4, device=DEV)
    kr[0, 0, 77, 3] = float("nan")
    q = synth.retrieval_queries(1, B, Hq, G, D, seed=4, device=DEV)[0]
    f32 = torch.float32
    ws = dbg.alloc_workspace(dbg.score_workspace(B, Hq, S), DEV)
    dbg.score(q, kr, z(B, fill=S), G, 0.125, torch.zeros((B, Hq, S), device=DEV),
              torch.zeros((B, Hq), device=DEV), z(B, Hq, dt=torch.int64),
              torch.zeros((B, G, S), dtype=f32, device=DEV), ws, phases=dbg.SCORE_LOGITS)
    assert dbg.check_device_errors() == E_RANGE
