#!/usr/bin/env python
"""Benchmark of the SpeContext decode-step hot path (libspc on B200).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config B]

One "step" = spc_score (LOGITS) + spc_select (NORM, GROUP, top-k, diff) +
spc_sparse_decode_attn over all L layers, on one batch of synthetic input,
inputs resident in HBM (each step's queries are read in place), CUDA graphs of up to 32
consecutive steps (a device decode loop).  No L2 flush: three
address-distinct copies of the inputs (each > L2) are rotated step by step; the steps are
timed with CUDA events on the launching stream.

Prints ONE JSON line (rank 0).  Metric: decode throughput in tokens/s (= batch x N / step time)
at the BASELINE.json config (default: config B, DeepSeek-R1-Distill-Llama-8B shape, ctx 32K).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode step throughput (tokens/s) of the retrieval + sparse-attention hot path"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="A/B (single GPU; one replica per GPU for N>1, with config E "
                         "context-sharded over the N GPUs attached), C (B=16, growing 128K "
                         "context), D (KV in pinned host memory, B=4), E (context-sharded "
                         "alone) or R (the retrieval head's front-end, NEXT-1) or M (MLA sparse "
                         "attention, NEXT-3), O (Algorithm 2 at run time) or L (whole LLM decode steps, "
                         "NEXT-4); default B")
    ap.add_argument("--batch", type=int, default=1, help="config R: requests per step (<= 16)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded", action="store_true",
                    help="N > 1: skip the attached config-E context-sharded measurement")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (CPU, gloo): spawn / rendezvous / max over ranks")
    ap.add_argument("--kv-layout", default="token", choices=["token", "layer"],
                    help="config D host KV layout: token-major records (one contiguous record "
                         "per token) or layer-major [L][B][G][rows][D]")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def init_pg(dev=None):
    """The process group of a multi-rank run (NCCL on GPUs, gloo for --dry-run), created
    once per process; None at world size 1."""
    if dist_env()[2] == 1:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        if dev is not None:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    return dist


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks on this node
    (torch.distributed.run, rendezvous on 127.0.0.1) and exit with its status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dry_run(args):
    """--dry-run: the launch plumbing alone, on CPU (no GPU, no kernels): every rank joins the
    gloo group, takes the max of a per-rank time over ranks, and rank 0 prints the JSON line
    shape with n_gpus = world size (tests/test_bench_launch.py)."""
    import torch
    rank, _, world = dist_env()
    pg = init_pg()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if pg:
        pg.barrier()
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "dry_run": True,
                          "max_over_ranks": float(t.item()),
                          "config": {"workload": "dry run (launch plumbing only)"}}), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


GRAPH_STEPS = 32  # decode steps per CUDA graph in the timed loops


def kernel_timeline(replay, names):
    """Per-kernel time inside a replayed multi-step graph, from CUPTI kernel records
    (torch.profiler; not timed): the kernels of a step run as a chain (each launched early
    by PDL, starting its work when its predecessor ends), so a kernel's share is its end
    minus its predecessor's end; averaged over the steady steps.  names: substring -> label
    in chain order.  Returns {label: us} or None."""
    import warnings

    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                replay()
                torch.cuda.synchronize()
        ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                    if e.device_type == torch.autograd.DeviceType.CUDA)
        lab = []
        for a, b, n in ks:
            for key, label in names:
                if key in n:
                    lab.append((a, b, label))
                    break
        per = len(names)
        steps = len(lab) // per
        if steps < 4:
            return None
        acc = {label: 0.0 for _, label in names}
        for st in range(1, steps - 1):  # steady steps: a predecessor in the same graph
            for i in range(per):
                j = st * per + i
                acc[lab[j][2]] += (lab[j][1] - lab[j - 1][1]) / (steps - 2)
        return {k: round(v, 2) for k, v in acc.items()}
    except Exception as e:  # noqa: BLE001 -- informational only
        print(f"# kernel timeline unavailable: {type(e).__name__}: {e}", file=sys.stderr)
        return None


def warm_graphs(st, graphs):
    """Replay every captured step graph once, untimed, then reset the rolling selection
    state: a CUDA graph's first launch carries a one-time upload cost that is not part of a
    decode step (all timed steps are then steady-state launches)."""
    import torch
    for g in graphs:
        g.replay()
        st.parity ^= 1
    torch.cuda.synchronize()
    st.reset_state()


def traffic_of(key):
    """ncu DRAM bytes per launch recorded in profiles/traffic.json (None if absent)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(key)
    except Exception:
        return None


def workload_name(c, key):
    return (f"{key}: {c['name']} (L={c['L']}, Hq={c['Hq']}, G={c['G']}, d={c['D']}, "
            f"ctx={c['S']}, batch={c['B']}, k={c['k']})")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU baseline (oracle)
def oracle_step_sample(c, kr_h, qr_h, kc_h, vc_h, ql_h, groups, scale):
    """The CPU oracle (as it stands) on `groups` of the G KV groups of one config step:
    scoring O1-O6 for those groups' heads, top-k O7, attention O10 for all L layers."""
    import numpy as np

    import oracle
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    alpha = Hq // G
    for g in groups:
        heads = slice(g * alpha, (g + 1) * alpha)
        q = np.ascontiguousarray(qr_h[:, heads])
        kr = np.ascontiguousarray(kr_h[:, g:g + 1])
        _, _, _, gs = oracle.score(q, kr, [S] * B, 1, scale)
        idx, _, cnt, _ = oracle.topk(gs, [S] * B, k, force_last=True)
        for l in range(L):
            for b in range(B):
                for h in range(g * alpha, (g + 1) * alpha):
                    oracle.attn_head(ql_h[l, b, h], kc_h[l, b, 0], vc_h[l, b, 0],
                                     idx[b, 0, :cnt[b, 0]], scale)


def cpu_inputs(c, seed):
    from paper_2512_00722_b200 import synth
    B, G, Hq, D, S, L = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"]
    kr = synth.bf16_bits(synth.retrieval_keys(B, G, S, D, seed=seed))
    qr = synth.bf16_bits(synth.retrieval_queries(1, B, Hq, G, D, seed=seed)[0])
    ql = synth.bf16_bits(synth.llm_queries(1, L, B, Hq, D, seed=seed)[0])
    kc, vc = synth.llm_kv(L, B, 1, S, D, seed=seed)  # one group's KV serves every sampled group
    return kr, qr, synth.bf16_bits(kc), synth.bf16_bits(vc), ql


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


_REF = {}


def _ref_group(g):
    """One KV group of a config step through the unmodified C oracle (a pool worker)."""
    c, kr, qr, kc, vc, ql, scale = _REF["args"]
    oracle_step_sample(c, kr, qr, kc, vc, ql, [g], scale)
    return g


def run_cpu_baseline(c, key, budget_s=10.0):
    """The oracle on the box's host cores: one thread (a 10 s sample of KV groups, scaled to a
    full step) and nproc cores (full steps measured by `bench.py --impl reference` in a fresh
    process: the G groups of a step in parallel processes)."""
    import oracle
    oracle.build()
    kr, qr, kc, vc, ql = cpu_inputs(c, 20251201)
    scale = float.fromhex("0x1.6a09e6p-4") if c["D"] == 128 else 0.125
    t0 = time.perf_counter()
    done = 0
    while True:
        oracle_step_sample(c, kr, qr, kc, vc, ql, [done % c["G"]], scale)
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    el = time.perf_counter() - t0
    step_s = el / done * c["G"]  # `done` of G groups measured -> full-step time
    single = {"value": c["B"] / step_s, "unit": "tokens/s", "cores": 1, "kind": "oracle",
              "sample": f"{done} KV-group samples ({done / c['G']:.2f} config-{key} steps: scoring, "
                        f"top-k, attention over all {c['L']} layers) in {el:.1f} s, single-threaded "
                        f"C oracle, time per full step = elapsed x {c['G']}/{done}",
              "seconds": round(el, 2)}
    multi = None
    try:  # nproc leg in a fresh CUDA-free process (the pool forks)
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                            "--config", key, "--steps", "3", "--warmup", "1"],
                           capture_output=True, text=True, timeout=300, cwd=ROOT)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
        multi = json.loads(line)["cpu_baseline"]
    except Exception as e:  # noqa: BLE001
        multi = {"error": f"{type(e).__name__}: {e}"[:200]}
    out = dict(multi) if multi and "value" in multi else dict(single)
    out["single_core"] = single
    out["host_cpu"] = host_cpu_model()
    out["nproc"] = os.cpu_count()
    return out


def bench_reference(args):
    """--impl reference: the CPU oracle as the reference arm (tier framing).  Every step is a
    FULL config step, measured: the G KV groups (independent problems) run in parallel
    processes of the unmodified single-threaded C oracle on the box's host cores."""
    import multiprocessing
    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_2512_00722_b200 import synth
    import oracle
    key = args.config
    c = synth.CONFIGS[key]
    oracle.build()
    kr, qr, kc, vc, ql = cpu_inputs(c, 20251201)
    scale = float.fromhex("0x1.6a09e6p-4") if c["D"] == 128 else 0.125
    _REF["args"] = (c, kr, qr, kc, vc, ql, scale)
    workers = max(1, min(os.cpu_count() or 1, c["G"]))
    times = []
    with multiprocessing.get_context("fork").Pool(workers) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_group, range(c["G"]), chunksize=1)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    step_s = statistics.mean(times)
    val = c["B"] / step_s
    sample = (f"every KV group of a config-{key} step (scoring, top-k, attention over all "
              f"{c['L']} layers), the {c['G']} groups in {workers} parallel processes of the "
              f"single-threaded C oracle; measured full steps (one group's KV serves every group: "
              f"host memory); host: {host_cpu_model()}, nproc {os.cpu_count()}")
    print(json.dumps({
        "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": workload_name(c, key)},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": workers, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ GPU
def bench_ours(args, attach=None):
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import roofline, spc, synth
    from paper_2512_00722_b200.pipeline import DecodeStep

    rank, local, world = dist_env()
    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        if rank == 0:
            spc_build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = init_pg(dev)
    key = args.config
    c = synth.CONFIGS[key]
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    seed = synth.BASE_SEED + 17 * rank
    nsteps = args.warmup + args.steps
    kr = synth.retrieval_keys(B, G, S, D, seed=seed, device=dev)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=seed, device=dev)
    qr = synth.retrieval_queries(nsteps + 1, B, Hq, G, D, seed=seed, device=dev)
    ql = synth.llm_queries(2, L, B, Hq, D, seed=seed, device=dev)
    seq = torch.full((B,), S, dtype=torch.int32, device=dev)
    st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
    # L2 policy: no flush; NSETS address-distinct copies of the inputs are rotated step by
    # step, so each step's reads (> L2 size) never find the previous steps' lines in L2.
    NSETS = 3
    copies = []
    for _ in range(NSETS - 1):
        kr2, kc2, vc2 = kr.clone(), kc.clone(), vc.clone()
        copies.append((kr2, kc2, vc2))
        st.add_input_set(kr2, [kc2[l] for l in range(L)], [vc2[l] for l in range(L)])
    set_bytes = kr.numel() * 2 + kc.numel() * 2 * 2

    # eager warm-up (sets kernel attributes), then the run as CUDA graphs of consecutive
    # decode steps (the warm-up steps, then chunks of up to GRAPH_STEPS timed steps: a device
    # decode loop, no host work between its steps, so consecutive steps chain inside one
    # graph with no graph-launch boundary); each step reads its queries in place (inputs
    # resident in HBM, no staging copies)
    st.step(qr[0], ql[0])
    n0 = spc.launch_count()
    st.capture()  # the (set, parity) graphs used by the e2e measurement
    items = [(i % NSETS, qr[i], ql[i % 2]) for i in range(nsteps)]
    wb = [(0, args.warmup)] if args.warmup > 0 else []
    bounds = wb + [(j, min(j + GRAPH_STEPS, nsteps)) for j in range(args.warmup, nsteps, GRAPH_STEPS)]
    timed = list(range(len(wb), len(bounds)))
    seq_graphs = st.capture_sequence(items, bounds=bounds)
    launches_per_step = (spc.launch_count() - n0) // (2 * NSETS + nsteps)
    stream = torch.cuda.current_stream()
    warm_graphs(st, seq_graphs)

    def run_chunk(ci):
        seq_graphs[ci].replay()
        st.parity ^= (bounds[ci][1] - bounds[ci][0]) & 1

    if wb:
        run_chunk(0)  # the warm-up steps
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(timed) + 1)]
    ev[0].record(stream)
    for j, ci in enumerate(timed):
        run_chunk(ci)
        ev[j + 1].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    step_ms = [ev[j].elapsed_time(ev[j + 1]) / (bounds[ci][1] - bounds[ci][0])
               for j, ci in enumerate(timed) for _ in range(bounds[ci][1] - bounds[ci][0])]
    # per-kernel times inside one replayed chunk (after the timed region, untimed)
    in_graph = None
    if st.fused and not st.one_launch and st.desc is not None:
        in_graph = kernel_timeline(lambda: run_chunk(timed[0]), [
            ("logits_tma", "logits"), ("lg_finalize", "finalize"), ("select_kernel", "select"),
            ("attn_tma", "attention"), ("tma_merge", "merge")])
    t_ms = ev[0].elapsed_time(ev[-1])
    if pg:
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        t_ms = float(t.item())
    ms_per_step = t_ms / args.steps
    value = B * world * args.steps / (t_ms / 1e3)
    n_load_tot = int(st.n_load.sum().item())  # elastic reuse of the last timed step
    cnt_tot = int(st.cnt[st.parity ^ 1].sum().item())

    # ---- per-kernel breakdown: eager steps with events between the phases (same stream)
    phases = (["score_select", "attn"] if st.one_launch else
              ["logits", "select", "attn"] if st.fused else ["score", "topk", "diff", "attn"])
    acc = {p: 0.0 for p in phases}
    reps = max(3, min(args.steps, 12))
    for j in range(reps):
        st.use_set(j % NSETS)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(len(phases) + 1)]
        cur, prev = st.parity, st.parity ^ 1
        st.q_ret.copy_(qr[j])
        # a 2 ms spin first, so the host enqueues every phase before the GPU reaches them:
        # the events then time the kernels back to back, not the host's launch latency
        torch.cuda._sleep(4_000_000)
        e[0].record(stream)
        if st.one_launch:
            spc.score_select(st.q_ret, st.kr, st.seq_len, st.scale, k, st.head_max, st.head_sumfix,
                             st.gs, st.idx[cur], st.cnt[cur], st.idx[prev], st.cnt[prev],
                             st.load_tok, st.n_load, st.ws_ss, force_last=True)
        elif st.fused:
            spc.score(st.q_ret, st.kr, st.seq_len, G, st.scale, st.logits, st.head_max,
                      st.head_sumfix, st.gs, st.ws_score, phases=spc.SCORE_LOGITS)
            e[1].record(stream)
            spc.select(st.logits, st.head_max, st.seq_len, G, k, st.head_sumfix, st.gs,
                       st.idx[cur], st.cnt[cur], st.idx[prev], st.cnt[prev], st.load_tok,
                       st.n_load, force_last=True)
        else:
            spc.score(st.q_ret, st.kr, st.seq_len, G, st.scale, st.logits, st.head_max,
                      st.head_sumfix, st.gs, st.ws_score)
            e[1].record(stream)
            spc.topk(st.gs, st.seq_len, k, st.idx[cur], st.cnt[cur], st.ws_topk,
                     force_last=True)
            e[2].record(stream)
            spc.elastic_diff(st.idx[prev], st.cnt[prev], st.idx[cur], st.cnt[cur],
                             st.load_tok, st.n_load)
        e[-2].record(stream)
        spc.sparse_decode_attn_kv(st.desc, st.q_llm, spc.KV_INDEXED, st.idx[cur], st.cnt[cur], k,
                                  st.scale, st.out, st.lse, st.ws_attn)
        e[-1].record(stream)
        torch.cuda.synchronize()
        for i, p in enumerate(phases):
            acc[p] += e[i].elapsed_time(e[i + 1]) / reps
        st.parity ^= 1
    attn_bytes = roofline.attn_bytes([S] * B, L, G, D, k)
    score_bytes = roofline.score_bytes([S] * B, G, D)
    step_bytes = attn_bytes + score_bytes
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # the attention's average launch duration as it runs inside the step (PDL-chained behind
    # the previous launch): 4 x NSETS launches back to back in one CUDA graph over the
    # rotating address-distinct input sets (each launch reads 256 MiB of KV > L2), CUDA events
    # around the replays on the launching stream; the eager per-phase times above include
    # each launch's full start-up (an event between kernels breaks the PDL overlap)
    p_last = st.parity ^ 1
    gs_ = torch.cuda.Stream()
    gs_.wait_stream(stream)
    ga = torch.cuda.CUDAGraph()
    n_attn = 4 * NSETS
    with torch.cuda.stream(gs_):
        with torch.cuda.graph(ga, stream=gs_):
            for r in range(n_attn):
                spc.sparse_decode_attn_kv(st.sets[r % NSETS][4], st.q_llm, spc.KV_INDEXED,
                                          st.idx[p_last], st.cnt[p_last], k, st.scale, st.out,
                                          st.lse, st.ws_attn, stream=gs_)
    stream.wait_stream(gs_)
    for _ in range(2):
        ga.replay()
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(3):
        ga.replay()
    eb.record(stream)
    torch.cuda.synchronize()
    attn_b2b_ms = ea.elapsed_time(eb) / (3 * n_attn)
    achieved = attn_bytes / (attn_b2b_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("attn", None)
        except Exception:
            traffic = None

    # ---- end to end through the public call with pinned host buffers; the retrieval
    # queries evolve step by step (the same AR(1) sequence as the device-resident run)
    q_ret_all = qr.cpu().pin_memory()
    q_ret_h = q_ret_all[1]
    q_llm_h = ql[0].cpu().pin_memory()
    out_h = torch.empty(st.out.shape, dtype=torch.float32).pin_memory()
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    bi = bo = 0
    nq = q_ret_all.shape[0]
    for j in range(max(args.warmup, 2 * NSETS)):  # untimed: every (set, parity) graph once
        st.use_set(j % NSETS)
        st.step_host(q_ret_all[j % nq], q_llm_h, out_h, use_graph=True)
    st.sync_host()
    torch.cuda.synchronize()
    e2[0].record(stream)
    for j in range(args.steps):
        st.use_set(j % NSETS)
        bi, bo = st.step_host(q_ret_all[(args.warmup + j) % nq], q_llm_h, out_h, use_graph=True)
    st.sync_host()  # the last step's read-back is inside the timed region
    e2[1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = e2[0].elapsed_time(e2[1])
    if pg:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = B * world * args.steps / (e2e_ms / 1e3)

    # ---- the same step started from token ids: the retrieval head's front-end (NEXT-1,
    # spc_rethead_qk at the Llama-3-8B retrieval-head shape, random-init weights) writes the
    # query and the newest key first; device-resident and end to end (host token ids in,
    # attention output back)
    fe = None
    if key == "B":
        from paper_2512_00722_b200 import rope
        V, H = 128256, 4096
        emb, norm_w, w_qk = synth.retrieval_head_weights(V, H, Hq, G, D, seed, device=dev)
        inv, msc = rope.yarn_inv_freq(D, factor=64.0, orig_ctx=2048)
        st.set_frontend(emb, norm_w, w_qk, torch.from_numpy(inv).to(dev), msc)
        toks = synth.tokens(args.steps, B, V, seed, device=dev)
        st.step(use_graph=False)
        st.capture()
        for j in range(args.warmup):
            st.use_set(j % NSETS)
            st.step(use_graph=True)
        torch.cuda.synchronize()
        e3 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e3[0].record(stream)
        for j in range(args.steps):
            st.use_set(j % NSETS)
            st.tokens[st.parity].copy_(toks[j], non_blocking=True)
            st.step(use_graph=True)
        e3[1].record(stream)
        torch.cuda.synchronize()
        fe_ms = e3[0].elapsed_time(e3[1]) / args.steps
        tok_h = toks.cpu().pin_memory()
        e3[0].record(stream)
        for j in range(args.steps):
            st.use_set(j % NSETS)
            fbi, fbo = st.step_host(tok_h[j], q_llm_h, out_h, use_graph=True)
        st.sync_host()
        e3[1].record(stream)
        torch.cuda.synchronize()
        fe_e2e_ms = e3[0].elapsed_time(e3[1]) / args.steps
        fe = {"what": "step incl. the retrieval head's front-end (spc_rethead_qk: token ids -> "
                      "query + newest key; NEXT-1)",
              "us_per_step": fe_ms * 1e3, "tokens_per_s": B / (fe_ms * 1e-3),
              "e2e_tokens_per_s": B / (fe_e2e_ms * 1e-3), "e2e_h2d_bytes_per_step": fbi,
              "e2e_d2h_bytes_per_step": fbo}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(c, key)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded; DESIGN.md §5)",
            "config": {"workload": workload_name(c, key),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": (f"inputs larger than L2: {NSETS} address-distinct copies of the "
                              f"inputs ({set_bytes / 2**30:.2f} GiB each) rotated step by step; "
                              "each step reads > 320 MiB"),
                       "kv_mode": "INDEXED (selected rows read in place)",
                       "graphs": f"CUDA graphs of up to {GRAPH_STEPS} consecutive decode steps",
                       "algorithmic_bytes_per_step": step_bytes,
                       "step_us_p50": statistics.median(step_ms) * 1e3,
                       "hbm_roofline_frac_step": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
                       "phase_us_in_graph": in_graph,
                       "phase_us_in_graph_how": ("CUPTI kernel records of one replayed chunk: "
                                                 "a kernel's end minus its predecessor's end"),
                       "phase_us": {p: round(acc[p] * 1e3, 2) for p in phases},
                       "phase_us_how": "eager, events between the phases (no PDL overlap)",
                       "attn_us_back_to_back": round(attn_b2b_ms * 1e3, 2),
                       "elastic_reuse": round(1 - n_load_tot / max(1, cnt_tot), 4),
                       "n_load_last_step": n_load_tot, "with_frontend": fe},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "attn_tma_kernel + tma_merge_kernel (spc_sparse_decode_attn_kv, all layers)",
                         "algorithmic_bytes_per_launch": attn_bytes,
                         "duration": "average launch, back to back in a CUDA graph (config."
                                     "attn_us_back_to_back); eager alone: phase_us.attn",
                         "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": bi,
                    "d2h_bytes_per_step": bo},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        if attach:
            line["config"].update(attach)
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()


def bench_sharded(args, embedded=False):
    """Config E: one 1M-token context sharded over the N ranks (t mod N), NCCL collectives.
    embedded: return the measurement (rank 0) instead of printing the JSON line."""
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import dist as sdist
    from paper_2512_00722_b200 import roofline, spc, synth

    rank, local, world = dist_env()
    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        if rank == 0:
            spc_build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tdist = init_pg(dev)
    key = "E"
    c = synth.CONFIGS[key]
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    P = world
    S_loc = sdist.local_len(S, P, rank)
    nsteps = args.warmup + args.steps
    seed = synth.BASE_SEED + 1000 + rank
    kr = synth.retrieval_keys(B, G, S_loc, D, seed=seed, device=dev)  # this rank's shard
    kc, vc = synth.llm_kv(L, B, G, S_loc, D, seed=seed, device=dev)
    qr = synth.retrieval_queries(nsteps + 1, B, Hq, G, D, seed=synth.BASE_SEED, device=dev)
    ql = synth.llm_queries(1, L, B, Hq, D, seed=synth.BASE_SEED, device=dev)[0]
    scale = float(torch.tensor(1.0 / math.sqrt(D), dtype=torch.float32))
    st = sdist.ShardState(rank, P, [S], kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)],
                          qr[0].clone(), ql, k, scale)
    ops = sdist.SpcOps()

    def body():
        if tdist is not None:
            return sdist.run_distributed(ops, st)
        sel, out, lse = sdist.run_emulated(ops, [st])
        return sel[0][0], sel[0][1], out, lse

    for i in range(args.warmup):
        st.q_ret.copy_(qr[i])
        body()
    torch.cuda.synchronize()
    graph = None
    n0 = spc.launch_count()
    try:
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                res = body()
        torch.cuda.current_stream().wait_stream(s)
        graph = g
    except Exception as e:  # NCCL capture unsupported here: time eager steps instead
        graph = None
        if rank == 0:
            print(f"# graph capture failed ({type(e).__name__}); timing eager steps", file=sys.stderr)
    launches_per_step = spc.launch_count() - n0
    stream = torch.cuda.current_stream()
    if tdist is not None:
        tdist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for j in range(args.steps):
        st.q_ret.copy_(qr[args.warmup + j])
        if graph is not None:
            graph.replay()
        else:
            res = body()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    t_ms = e0.elapsed_time(e1)
    if tdist is not None:
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        t_ms = float(t.item())
    ms_per_step = t_ms / args.steps
    value = B * args.steps / (t_ms / 1e3)
    # e2e: the same step with the retrieval query copied from pinned host memory and the
    # merged attention output read back to pinned host memory every step
    q_h = qr[1].cpu().pin_memory()
    out_h = torch.empty(res[2].shape, dtype=res[2].dtype).pin_memory()
    if tdist is not None:
        tdist.barrier()
    torch.cuda.synchronize()
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e2[0].record(stream)
    for j in range(args.steps):
        st.q_ret.copy_(q_h, non_blocking=True)
        if graph is not None:
            graph.replay()
        else:
            res = body()
        out_h.copy_(res[2], non_blocking=True)
    e2[1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = e2[0].elapsed_time(e2[1])
    if tdist is not None:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": B * args.steps / (e2e_ms / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": q_h.numel() * q_h.element_size(),
           "d2h_bytes_per_step": out_h.numel() * out_h.element_size()}
    cnt_loc = int(res[1].sum().item())
    rank_bytes = S_loc * G * D * 2 + cnt_loc * L * D * 2 * 2
    if launches_per_step == 0:
        launches_per_step = 8
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = rank_bytes / (ms_per_step * 1e-3) / 1e9
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded per rank; DESIGN.md §5)",
            "config": {"workload": workload_name(c, key), "parallelism": f"context-sharded x{P}",
                       "l2": "inputs larger than L2 (each step streams > 2 GiB / P per rank)",
                       "graph": graph is not None,
                       "rank0_bytes_per_step": rank_bytes},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "whole sharded step on rank 0 (all kernels + collectives)",
                         "algorithmic_bytes_per_launch": rank_bytes},
            "cpu_baseline": None,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        if not embedded:
            print(json.dumps(line), flush=True)
    if tdist is not None:
        tdist.barrier()
    del st, kr, kc, vc
    torch.cuda.empty_cache()
    return line


def bench_grow(args):
    """Config C: B = 16 requests at 131,072 tokens, the context growing by one token per step
    (seq_len += 1 inside the timed loop; the new rows are pre-written).  The LLM KV of the 32
    layers is 8 physical layers: layer l reads physical layer l mod 8 at a row offset of
    (l // 8) x 1024 rows, so concurrently processed layers never touch the same lines and
    every step still reads its selected rows from HBM (73 GB of KV resident)."""
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import roofline, spc, synth
    from paper_2512_00722_b200.pipeline import DecodeStep

    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        spc_build.build()
    dev = torch.device("cuda", 0)
    c = synth.CONFIGS["C"]
    B, G, Hq, D, S0, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    PHYS, OFF = 8, 1024
    nsteps = args.warmup + args.steps
    Smax = (S0 + nsteps + 3) // 4 * 4
    rows = Smax + (L // PHYS - 1) * OFF
    seed = synth.BASE_SEED + 3
    kr = synth.retrieval_keys(B, G, Smax, D, seed=seed, device=dev)
    kv = [synth.llm_kv(1, B, G, rows, D, seed=seed + 11 * p, device=dev) for p in range(PHYS)]
    k_layers = [kv[l % PHYS][0][0].view(-1)[(l // PHYS) * OFF * D:] for l in range(L)]
    v_layers = [kv[l % PHYS][1][0].view(-1)[(l // PHYS) * OFF * D:] for l in range(L)]
    qr = synth.retrieval_queries(nsteps + 1, B, Hq, G, D, seed=seed, device=dev)
    ql = synth.llm_queries(2, L, B, Hq, D, seed=seed, device=dev)
    seq = torch.full((B,), S0, dtype=torch.int32, device=dev)
    st = DecodeStep(kr, k_layers, v_layers, seq, L, Hq, k, kv_rows=rows,
                    fused=None if os.environ.get("SPC_FUSED") is None else os.environ["SPC_FUSED"] == "1")
    st.step(qr[0], ql[0])
    n0 = spc.launch_count()
    seq_graphs = st.capture_sequence([(0, qr[i], ql[i % 2]) for i in range(nsteps)])
    launches_per_step = (spc.launch_count() - n0) // nsteps
    warm_graphs(st, seq_graphs)
    seq.fill_(S0)
    stream = torch.cuda.current_stream()

    def one_step(i):
        seq.add_(1)  # the step's new token (its rows are already in the caches)
        seq_graphs[i].replay()  # the step's queries are read in place
        st.parity ^= 1

    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    n_load, cnt = [], []
    ev[0].record(stream)
    for j in range(args.steps):
        one_step(args.warmup + j)
        ev[j + 1].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    n_load.append(int(st.n_load.sum().item()))
    cnt.append(int(st.cnt[st.parity ^ 1].sum().item()))
    step_ms = [ev[j].elapsed_time(ev[j + 1]) for j in range(args.steps)]
    t_ms = ev[0].elapsed_time(ev[-1])
    ms = t_ms / args.steps
    S_mid = S0 + args.warmup + args.steps // 2
    step_bytes = roofline.step_bytes([S_mid] * B, L, G, D, k)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = step_bytes / (ms * 1e-3) / 1e9
    print(json.dumps({
        "metric": METRIC, "value": B / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded; DESIGN.md §5)",
        "config": {"workload": workload_name(c, "C") + ", +1 token per step",
                   "ctx_range": [S0 + args.warmup + 1, S0 + nsteps],
                   "kv": f"{PHYS} physical layers aliased (row offset {OFF} per alias), "
                         f"{sum(t.numel() for p in kv for t in p) * 2 / 2**30:.1f} GiB",
                   "l2": "working set 73 GB >> L2; aliased layers read at distinct rows",
                   "algorithmic_bytes_per_step": step_bytes,
                   "step_us_p50": statistics.median(step_ms) * 1e3,
                   "step_us_p10_p90": [sorted(step_ms)[len(step_ms) // 10] * 1e3,
                                       sorted(step_ms)[(9 * len(step_ms)) // 10] * 1e3],
                   "fused_select": st.fused,
                   "elastic_reuse_last_step": round(1 - n_load[-1] / max(1, cnt[-1]), 4),
                   "n_load_last_step": n_load[-1]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "whole step (LOGITS + select + attention)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }), flush=True)


def bench_offload(args):
    """Config D (offloaded KV): S = 262,144, k = 2048, the LLM KV in pinned host memory,
    SLOTS mode: each step spc_gather_kv copies only the newly selected rows (elastic load)
    over PCIe into the HBM budget buffers, then attention reads the buffers.  Host RAM on
    the box (196 GB) cannot hold config D's 1.1 TB of KV, so B = 8 requests by default
    (--batch; per-request traffic is unchanged, bytes scale with B) over 8 physical layers
    aliased at distinct row offsets (70 GB pinned at B = 8).  Reports the PCIe bytes moved
    per step against the measured pinned host->device copy bandwidth, and the same step with
    the asynchronous prefetch dataflow: the gather of layer group j on a side
    stream overlapping the attention of group j-1 (4 groups of 8 layers = whole 4 KiB
    records), with the fraction of the attention hidden under the gather."""
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import spc, synth
    from paper_2512_00722_b200.pipeline import DecodeStep

    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        spc_build.build()
    dev = torch.device("cuda", 0)
    c = synth.CONFIGS["D"]
    B = args.batch if args.batch > 1 else 8
    G, Hq, D, S, L, k = c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    PHYS, OFF = 8, 1024
    nsteps = args.warmup + args.steps
    rows = S + (L // PHYS - 1) * OFF
    seed = synth.BASE_SEED + 4
    kr = synth.retrieval_keys(B, G, S, D, seed=seed, device=dev)
    token_major = args.kv_layout == "token"
    src_strides = None
    if token_major:
        # one record per token: [PHYS layers][K, V][D] (4 KiB); layer l reads physical layer
        # l % PHYS of the record of token t + (l // PHYS) * OFF (a real deployment's record
        # holds all L layers: 16 KiB contiguous per selected token -- this is conservative)
        rec = torch.empty((B, G, rows, PHYS, 2, D), dtype=torch.bfloat16, pin_memory=True)
        for b in range(B):
            for g in range(G):
                rec[b, g].copy_(synth.normal_bf16((rows, PHYS, 2, D), seed * 131 + b * G + g,
                                                  device=dev))
        host = [[rec]]
        k_src = [rec[:, :, (l // PHYS) * OFF:, l % PHYS, 0] for l in range(L)]
        v_src = [rec[:, :, (l // PHYS) * OFF:, l % PHYS, 1] for l in range(L)]
        src_strides = (PHYS * 2 * D, rows * PHYS * 2 * D)
    else:
        host = []
        for p in range(PHYS):  # generated on the GPU layer by layer, copied into pinned memory
            pair = []
            for t in range(2):
                h = torch.empty((B, G, rows, D), dtype=torch.bfloat16, pin_memory=True)
                for b in range(B):
                    h[b].copy_(synth.normal_bf16((G, rows, D), seed * 131 + p * 7 + t * 3 + b,
                                                 device=dev))
                pair.append(h)
            host.append(pair)
        k_src = [host[l % PHYS][0].view(-1)[(l // PHYS) * OFF * D:] for l in range(L)]
        v_src = [host[l % PHYS][1].view(-1)[(l // PHYS) * OFF * D:] for l in range(L)]
    kb = torch.zeros((L, B, G, k, D), dtype=torch.bfloat16, device=dev)
    vb = torch.zeros_like(kb)
    qr = synth.retrieval_queries(nsteps + 1, B, Hq, G, D, seed=seed, device=dev)
    ql = synth.llm_queries(2, L, B, Hq, D, seed=seed, device=dev)
    seq = torch.full((B,), S, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def measure(groups):
        """(ms per step, rows loaded per step, launches per step, clocks, step object)"""
        kb.zero_()
        vb.zero_()
        st = DecodeStep(kr, [kb[l] for l in range(L)], [vb[l] for l in range(L)], seq, L, Hq, k,
                        mode="slots", k_src_layers=k_src, v_src_layers=v_src, kv_rows=k,
                        src_rows=rows, src_strides=src_strides, prefetch_groups=groups)
        st.step(qr[0], ql[0])
        n0 = spc.launch_count()
        seq_graphs = st.capture_sequence([(0, qr[i], ql[i % 2]) for i in range(nsteps)])
        per_step = (spc.launch_count() - n0) // nsteps
        warm_graphs(st, seq_graphs)
        kb.zero_()
        vb.zero_()
        loaded = torch.zeros((), dtype=torch.int64, device=dev)

        def one_step(i):
            seq_graphs[i].replay()
            st.parity ^= 1
            loaded.add_(st.n_load.sum())

        for i in range(args.warmup):
            one_step(i)
        torch.cuda.synchronize()
        loaded.zero_()
        sampler = ClockSampler(0)
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for j in range(args.steps):
            one_step(args.warmup + j)
        e1.record(stream)
        torch.cuda.synchronize()
        clk = sampler.stop()
        return e0.elapsed_time(e1) / args.steps, int(loaded.item()) / args.steps, per_step, clk, st

    ms, rows_loaded, launches_per_step, clocks, st = measure(1)
    ms_pipe, _, launches_pipe, clocks_pipe, st_pipe = measure(4)
    # attention alone over the filled budget buffers (all layers), for the overlap fraction
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        a0.record(stream)
        for _ in range(10):
            st_pipe._attn_slots(st_pipe.last, st_pipe.q_llms[0], st_pipe.outs[0], st_pipe.lses[0],
                                0, L, stream)
        a1.record(stream)
        torch.cuda.synchronize()
    attn_ms = a0.elapsed_time(a1) / 10
    overlap = max(0.0, min(1.0, (ms - ms_pipe) / attn_ms)) if attn_ms > 0 else 0.0
    pcie_bytes = rows_loaded * L * 2 * D * 2
    # denominator: pinned host -> device copy of 1 GiB
    hsrc = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    ddst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    ddst.copy_(hsrc, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(3):
        ddst.copy_(hsrc, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    h2d = 3 * (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9
    achieved = pcie_bytes / (ms * 1e-3) / 1e9
    print(json.dumps({
        "metric": METRIC, "value": B / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded; DESIGN.md §5)",
        "config": {"workload": workload_name(dict(c, B=B), "D") + " (B reduced from 32: host RAM of the box)",
                   "kv": (f"LLM KV in pinned host memory, token-major records [{PHYS} layers][K,V]"
                          f"[D] (4 KiB) per token, layer l = physical l % {PHYS} of the record "
                          f"of token t + (l // {PHYS}) * {OFF}" if token_major else
                          f"LLM KV in pinned host memory, layer-major: {PHYS} physical layers "
                          f"aliased at row offsets") +
                         f", {sum(t.numel() for p in host for t in p) * 2 / 2**30:.1f} GiB",
                   "kv_mode": ("SLOTS: spc_gather_kv_strided of the new tokens' records"
                               if token_major else "SLOTS: spc_gather_kv of the new rows") +
                              " (host -> HBM budget buffers, zero-copy reads of pinned memory),"
                              " then attention",
                   "rows_loaded_per_step": rows_loaded,
                   "elastic_reuse": round(1 - rows_loaded / (B * G * k), 4),
                   "pcie_bytes_per_step": pcie_bytes,
                   "pinned_h2d_copy_gbs": round(h2d, 1),
                   "prefetch_pipeline": {
                       "what": "gather of layer group j (8 layers) on a prefetch stream, "
                               "attention of group j waiting on its event (P:350, P:374)",
                       "groups": 4, "ms_per_step": ms_pipe, "serial_ms_per_step": ms,
                       "attention_alone_ms": attn_ms,
                       "attention_hidden_frac": round(overlap, 3),
                       "pcie_gbs": round(pcie_bytes / (ms_pipe * 1e-3) / 1e9, 1),
                       "tokens_per_s": B / (ms_pipe * 1e-3), "gpu_launches_per_step": launches_pipe,
                       "clocks": clocks_pipe}},
        "roofline": {"bound": "pcie", "achieved": achieved, "peak": h2d, "unit": "GB/s",
                     "frac": achieved / h2d, "traffic": None,
                     "kernel": "whole step, PCIe bytes of the elastic gather / step time",
                     "peak_source": "measured pinned host->device cudaMemcpy of 1 GiB"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }), flush=True)


def bench_alg2(args):
    """Algorithm 2 at run time (NEXT-2): the config-B shape (32 layers, ctx 32K,
    k 2048) with the planner's thresholds for a GPU-memory budget that forces n of the 32
    layers' KV off the GPU at this context; n in {0, 8, 16, 32}: the offloads (Algorithm 2's
    KV_Cache_Offload, once per layer), then the steady-state mixed step -- resident layers
    attended in place, offloaded layers through the elastic PCIe gather of their new rows
    into HBM budget buffers -- timed as CUDA graphs."""
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import spc, synth
    from paper_2512_00722_b200.offload import OffloadingDecodeStep

    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        spc_build.build()
    dev = torch.device("cuda", 0)
    c = synth.CONFIGS["B"]
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    seed = synth.BASE_SEED + 7
    qr = synth.retrieval_queries(args.warmup + args.steps + 2, B, Hq, G, D, seed=seed, device=dev)
    ql = synth.llm_queries(2, L, B, Hq, D, seed=seed, device=dev)
    stream = torch.cuda.current_stream()
    rows = []
    layer_counts = [int(x) for x in os.environ.get("SPC_O_LAYERS", "0,8,16,32").split(",")]
    # the first configuration of the process runs twice, the first pass discarded: a fresh
    # process's first graphs measured 6x slower (0.75 vs 0.12 ms at n = 0)
    for n in [layer_counts[0]] + layer_counts:
        kr = synth.retrieval_keys(B, G, S, D, seed=seed, device=dev)
        kv = synth.llm_kv(L, B, G, S, D, seed=seed, device=dev)
        k_layers = [kv[0][l].clone() for l in range(L)]  # one allocation per layer
        v_layers = [kv[1][l].clone() for l in range(L)]
        del kv
        torch.cuda.synchronize()
        hbm0 = torch.cuda.memory_allocated(dev)
        # the planner (Eq. 7, Algorithm 1) for the budget of L - n resident layers at S + 1
        cfg = spc.plan_cfg(1, 0, L, G, D, 1, B, extra_layers=1, runtime_factor=0.0)
        cfg.mem_gpu = spc.plan_mem_part(cfg, S + 1, L - n)  # S^T_n = S + 1 > S (R27)
        th = spc.plan_thresholds(cfg)
        seq = torch.full((B,), S, dtype=torch.int32, device=dev)
        st = OffloadingDecodeStep(kr, k_layers, v_layers, seq, L, Hq, k, th)
        del k_layers, v_layers
        st.step(qr[0], ql[0], S)  # Algorithm 2 offloads n layers before this step
        torch.cuda.synchronize()
        assert st.l_cpu == n, (n, st.l_cpu)
        freed = hbm0 - torch.cuda.memory_allocated(dev)
        mig = [m[2] for m in st.migrations]
        # one graph per step of an evolving query sequence (the AR(1) retrieval queries: each
        # step selects ~19% new rows, which the offloaded layers gather over PCIe)
        nst = args.warmup + args.steps
        graphs = st.capture([(qr[1 + i], ql[i % 2]) for i in range(nst)], S)
        torch.cuda._sleep(400_000_000)  # ~0.2 s busy: clocks up before a ~ms timed window
        for i in range(args.warmup):
            graphs[i].replay()
        torch.cuda.synchronize()
        loaded = torch.zeros((), dtype=torch.int64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            graphs[args.warmup + i].replay()
            loaded.add_(st.n_load.sum())
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        rows_loaded = int(loaded.item()) / args.steps
        rows.append({"offloaded_layers": n, "resident_layers": L - n, "ms_per_step": ms,
                     "tokens_per_s": B / (ms * 1e-3),
                     "thresholds_head": [int(x) for x in th[: min(len(th), n + 2)]],
                     "hbm_bytes_released": int(freed),
                     "offload_seconds_per_layer": (sum(mig) / len(mig)) if mig else None,
                     "pcie_bytes_per_step": rows_loaded * n * 2 * D * 2})
        del st, graphs, kr
        torch.cuda.empty_cache()
    rows = rows[1:]
    base = rows[0]
    print(json.dumps({
        "metric": METRIC, "value": base["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": base["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded; DESIGN.md §5)",
        "config": {"workload": "O: Algorithm 2 at run time on the config-B shape (L=32, Hq=32, "
                               f"G=8, d=128, ctx={S}, batch={B}, k={k}); n layers offloaded by "
                               "the planner's thresholds, the rest resident",
                   "mixed_steps": rows,
                   "note": "value / ms_per_step: n = 0 (all resident); the offloaded layers' "
                           "rows are gathered over PCIe every step (elastic load)"},
        "roofline": None, "gpu_launches": None,
    }), flush=True)


def bench_frontend(args):
    """Config R: the retrieval head's front-end spc_rethead_qk at the
    config-B retrieval-head shape (Llama-3-8B: vocabulary 128,256, hidden 4,096, 32 query /
    8 key heads of 128, YaRN x64 over a 2k original context), random-init weights.  Step =
    one token per request: embedding -> RMSNorm -> Q/K projection (40 MiB of bf16 weights)
    -> RoPE -> K append.  HBM-bound GEMV: roofline bytes = weights + embedding rows + writes.
    Four address-distinct weight copies (160 MiB > L2) are rotated launch by launch, in a CUDA
    graph of 4 launches."""
    import torch

    import oracle
    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import rope, spc, synth

    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        spc_build.build()
    dev = torch.device("cuda", 0)
    B, V, H, Hq, G, D = args.batch, 128256, 4096, 32, 8, 128
    Smax, NC = 32768 + 64, 4
    seed = synth.BASE_SEED + 5
    emb, norm_w, w0 = synth.retrieval_head_weights(V, H, Hq, G, D, seed, device=dev)
    ws = [w0] + [w0.clone() for _ in range(NC - 1)]
    inv, mscale = rope.yarn_inv_freq(D, factor=64.0, orig_ctx=2048)
    inv_d = torch.from_numpy(inv).to(dev)
    toks = synth.tokens(NC, B, V, seed, device=dev)
    pos = torch.full((B,), 32768, dtype=torch.int32, device=dev)
    q = torch.zeros((B, Hq, D), dtype=torch.bfloat16, device=dev)
    kr = torch.zeros((B, G, Smax, D), dtype=torch.bfloat16, device=dev)
    sl = torch.zeros(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream()

    def call(i, st=None):
        spc.rethead_qk(toks[i % NC], emb, norm_w, 1e-5, ws[i % NC], inv_d, mscale, pos, Hq, G,
                       q, kr, seq_len_out=sl, stream=st)

    with torch.cuda.stream(stream):
        for i in range(NC):
            call(i, stream)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = spc.launch_count()
        with torch.cuda.graph(g, stream=stream):
            for i in range(NC):
                call(i, stream)
        per_replay = spc.launch_count() - n0
        for _ in range(max(1, args.warmup)):
            g.replay()
        stream.synchronize()
        reps = max(1, args.steps // NC)
        sampler = ClockSampler(0)
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        stream.synchronize()
        clocks = sampler.stop()
    n_launch = reps * NC
    us = e0.elapsed_time(e1) * 1e3 / n_launch
    wbytes = (Hq + G) * D * H * 2
    alg = wbytes + B * H * 2 + B * (Hq + G) * D * 2
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg / (us * 1e-6) / 1e9
    # e2e through the public call: token ids and positions from pinned host memory, the
    # query read back, every step
    tok_h = toks.cpu().pin_memory()
    pos_h = pos.cpu().pin_memory()
    q_h = torch.empty(q.shape, dtype=q.dtype).pin_memory()
    tok_d = torch.empty_like(toks[0])
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(stream):
        e2[0].record(stream)
        for i in range(args.steps):
            tok_d.copy_(tok_h[i % NC], non_blocking=True)
            pos.copy_(pos_h, non_blocking=True)
            spc.rethead_qk(tok_d, emb, norm_w, 1e-5, ws[i % NC], inv_d, mscale, pos, Hq, G, q,
                           kr, seq_len_out=sl, stream=stream)
            q_h.copy_(q, non_blocking=True)
        e2[1].record(stream)
        stream.synchronize()
    e2e_us = e2[0].elapsed_time(e2[1]) * 1e3 / args.steps
    # CPU baseline: the oracle's front-end (C, fp64 projection) on one request
    import time
    oracle.build()
    wh = synth.bf16_bits(w0)
    xh = synth.bf16_bits(emb[toks[0, :1].long()])
    nwh = synth.bf16_bits(norm_w)
    t0 = time.perf_counter()
    n_cpu = 0
    while time.perf_counter() - t0 < 3.0:
        xn = oracle.rmsnorm_bf16(xh, nwh, 1e-5)
        oracle.rethead_qk(wh, xn, inv, [32768], D, mscale=mscale)
        n_cpu += 1
    cpu_s = (time.perf_counter() - t0) / n_cpu
    print(json.dumps({
        "metric": METRIC, "value": B / (us * 1e-6), "unit": "tokens/s", "n_gpus": 1,
        "steps": n_launch, "warmup": args.warmup, "ms_per_step": us * 1e-3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded random-init retrieval-head weights; DESIGN.md §5)",
        "config": {"workload": f"R: retrieval-head front-end (NEXT-1), Llama-3-8B shape "
                               f"(V={V}, H={H}, Hq={Hq}, G={G}, d={D}), YaRN x64, batch={B}",
                   "l2": f"{NC} address-distinct weight copies ({NC * wbytes / 2**20:.0f} MiB > "
                         f"L2) rotated launch by launch",
                   "algorithmic_bytes_per_step": alg, "front_end_us": us},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_of("rethead_b1") if B == 1 else None,
                     "kernel": "rethead_kernel (spc_rethead_qk)",
                     "algorithmic_bytes_per_launch": alg,
                     "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)"},
        "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                         "sample": f"{n_cpu} single-request front-end calls of the C oracle "
                                   f"(RMSNorm + fp64 projection + RoPE) in {n_cpu * cpu_s:.1f} s"},
        "e2e": {"value": B / (e2e_us * 1e-6), "unit": "tokens/s", "h2d_bytes_per_step": B * 8,
                "d2h_bytes_per_step": B * Hq * D * 2},
        "gpu_launches": per_replay * reps,
        "clocks": clocks,
    }), flush=True)


def bench_mla(args):
    """Config M: MLA sparse decode attention over each head's selected
    latent rows (spc_mla_sparse_attn) at the DeepSeek-V2-Lite attention shape: 27 layers, 16
    heads, latent 512 + rope 64, no-rope / value head dims 128, 32K context, budget 2048
    per head, B = 1.  Selections are synthetic (sorted random rows per head: the retrieval
    that produces them is the head-level path measured by config B).  Step = one call for
    all 27 layers (2 launches); 3 address-distinct latent caches rotated (3.1 GB > L2)."""
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import spc, synth

    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        spc_build.build()
    dev = torch.device("cuda", 0)
    L, B, H, DN, DV, DC, DR, S, k, NS = 27, 1, 16, 128, 128, 512, 64, 32768, 2048, 3
    seed = synth.BASE_SEED + 6
    caches = [[synth.normal_bf16((B, S, DC + DR), seed + 97 * c + l, device=dev) for l in range(L)]
              for c in range(NS)]
    w_uk = [(synth.normal_bf16((H, DN, DC), seed + 1000 + l, device=dev, dtype=torch.float32)
             * DC ** -0.5).to(torch.bfloat16) for l in range(L)]
    w_uv = [(synth.normal_bf16((H, DV, DC), seed + 2000 + l, device=dev, dtype=torch.float32)
             * DC ** -0.5).to(torch.bfloat16) for l in range(L)]
    q = synth.normal_bf16((L, B, H, DN + DR), seed + 3000, device=dev)
    g = torch.Generator(device="cpu").manual_seed(seed)
    idx = torch.stack([torch.sort(torch.randperm(S, generator=g)[:k])[0] for _ in range(B * H)])
    idx = idx.view(B, H, k).to(torch.int32).to(dev)
    cnt = torch.full((B, H), k, dtype=torch.int32, device=dev)
    out = torch.zeros((L, B, H, DV), dtype=torch.float32, device=dev)
    ws = spc.alloc_workspace(spc.mla_workspace(L, B, H, k), dev)
    scale = (DN + DR) ** -0.5
    stream = torch.cuda.Stream()
    ctabs = [spc.ptr_table(caches[c], dev) for c in range(NS)]
    uktab, uvtab = spc.ptr_table(w_uk, dev), spc.ptr_table(w_uv, dev)

    def step(c, st):  # all 27 layers in one call
        spc.mla_sparse_attn(q, ctabs[c], uktab, uvtab, idx, cnt, S, DN, DV, scale, out, None, ws,
                            stream=st)

    graphs = []
    with torch.cuda.stream(stream):
        for c in range(NS):
            step(c, stream)
        stream.synchronize()
        n0 = spc.launch_count()
        for c in range(NS):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                step(c, stream)
            graphs.append(gr)
        per_step = (spc.launch_count() - n0) // NS
        for i in range(args.warmup):
            graphs[i % NS].replay()
        stream.synchronize()
        sampler = ClockSampler(0)
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            graphs[i % NS].replay()
        e1.record(stream)
        stream.synchronize()
        clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    alg = L * (B * H * k * (DC + DR) * 2 + H * (DN + DV) * DC * 2)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg / (ms * 1e-3) / 1e9
    print(json.dumps({
        "metric": METRIC, "value": B / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded latent caches, weights and per-head selections)",
        "config": {"workload": f"M: MLA sparse attention (NEXT-3), DeepSeek-V2-Lite attention "
                               f"shape (L={L}, H={H}, latent {DC}+{DR}, d_nope={DN}, d_v={DV}, "
                               f"ctx={S}, k={k} per head, batch={B})",
                   "l2": f"{NS} address-distinct latent caches rotated step by step",
                   "algorithmic_bytes_per_step": alg},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_of("mla_attn_27_layers"),
                     "traffic_note": "ncu DRAM bytes of mla_attn_kernel per step: below the "
                                     "per-head algorithmic bytes (heads sharing a selected "
                                     "latent row hit L2)",
                     "kernel": "mla_absorb_kernel + mla_attn_kernel, all layers",
                     "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)"},
        "gpu_launches": per_step * args.steps,
        "clocks": clocks,
    }), flush=True)


def bench_llm(args):
    """Config L: whole LLM decode steps around the hot path -- the
    DeepSeek-R1-Distill-Llama-8B shape (32 layers, hidden 4096, 32 q / 8 kv heads of 128,
    FFN 14336, vocabulary 128256; random bf16 weights, 15 GiB), ctx 32K growing by one token
    per step, k = 2048: the retrieval head once per step, then per layer RMSNorm, the QKV /
    O / gate-up / down projections (cuBLAS), RoPE + KV append, sparse attention over the
    selected rows (libspc), and the next token = argmax on the device.  Three variants, each
    one CUDA graph per step: (1) KV resident in HBM (INDEXED); (2) KV in pinned host memory
    with the elastic gathers serialised in front of each layer; (3) the same with the gathers
    on a prefetch stream overlapping the layers' dense compute (Fig. 3).
    B = --batch (default 4).  Inputs larger than L2: each step streams 15 GiB of weights."""
    import torch

    from paper_2512_00722_b200 import build as spc_build
    from paper_2512_00722_b200 import rope, spc, synth
    from paper_2512_00722_b200.llm import LlmDecoder

    if not os.path.exists(spc.LIB_PATH) or not spc_build.up_to_date():
        spc_build.build()
    dev = torch.device("cuda", 0)
    c = dict(synth.LLAMA8B)
    L, H, Hq, G, D, F, V = (c[x] for x in ("L", "H", "Hq", "G", "D", "F", "V"))
    B = args.batch if args.batch > 1 else 4
    S0, k = int(os.environ.get("SPC_L_CTX", "32768")), 2048
    nsteps = args.warmup + args.steps
    Smax = S0 + nsteps + 64
    seed = synth.BASE_SEED + 9
    w = synth.llm_weights(L, H, Hq, G, D, F, V, seed, device=dev)
    _, nw, w_qk = synth.retrieval_head_weights(V, H, Hq, G, D, seed, device=dev)
    inv_r, ms = rope.yarn_inv_freq(D, factor=64.0, orig_ctx=2048)
    ret = dict(emb=w["emb"], norm_w=nw, w_qk=w_qk, inv_freq=torch.from_numpy(inv_r).to(dev),
               mscale=ms)
    kr = synth.retrieval_keys(B, G, Smax, D, seed=seed, device=dev)
    kc, vc = synth.llm_kv(L, B, G, Smax, D, seed=seed, device=dev)
    tok0 = synth.tokens(1, B, V, seed, device=dev)[0]
    seq0 = torch.full((B,), S0 + 1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    results = {}

    def run(name, dec):
        seq = dec.seq_len
        dec.reset(tok0, seq0)
        dec.step()  # eager: kernel attributes, cuBLAS handles
        torch.cuda.synchronize()
        n0 = spc.launch_count()
        dec.capture()
        launches = (spc.launch_count() - n0) // 2
        dec.reset(tok0, seq0)
        for _ in range(args.warmup):
            dec.step(use_graph=True)
        torch.cuda.synchronize()
        out_tok = torch.empty((args.steps, B), dtype=torch.int32, pin_memory=True)
        loaded = torch.zeros((), dtype=torch.int64, device=dev)
        sampler = ClockSampler(0)
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for j in range(args.steps):
            t = dec.step(use_graph=True)
            out_tok[j].copy_(t, non_blocking=True)  # the generated token back to the host
            loaded.add_(dec.st.n_load.sum())
        e1.record(stream)
        torch.cuda.synchronize()
        clk = sampler.stop()
        ms = e0.elapsed_time(e1) / args.steps
        assert int(seq[0].item()) == S0 + 1 + args.warmup + args.steps
        results[name] = dict(ms_per_step=ms, tokens_per_s=B / (ms * 1e-3),
                             gpu_launches_per_step=launches, clocks=clk,
                             rows_loaded_per_step=int(loaded.item()) / args.steps)
        return ms

    seq = torch.empty_like(seq0)
    # the synthetic retrieval-query trace (AR(1) drift): the adjacent-step
    # similarity of a real trace, which a random-weight model's own queries lack
    trace = synth.retrieval_queries(nsteps + 2, B, Hq, G, D, seed=seed, device=dev)
    # the first measured configuration of a process runs slow (seen on configs O and L), so
    # the resident variant is run twice and the second run is kept
    for name, tq in (("resident", None), ("resident", None), ("resident_trace", trace)):
        dec = LlmDecoder(w, c, ret, kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)],
                         seq, k, kv="resident", trace_queries=tq)
        run(name, dec)
        wbytes = dec.weight_bytes()
        del dec
        torch.cuda.empty_cache()
    ms_res = results["resident"]["ms_per_step"]
    # offloaded: the LLM KV moved into pinned host memory layer by layer
    kh = [torch.empty((B, G, Smax, D), dtype=torch.bfloat16, pin_memory=True) for _ in range(L)]
    vh = [torch.empty_like(t, pin_memory=True) for t in kh]
    for l in range(L):
        kh[l].copy_(kc[l])
        vh[l].copy_(vc[l])
    del kc, vc
    torch.cuda.empty_cache()
    for name, pf, tq in (("offload_serial", False, None), ("offload_prefetch", True, None),
                         ("offload_serial_trace", False, trace),
                         ("offload_prefetch_trace", True, trace)):
        dec = LlmDecoder(w, c, ret, kr, kh, vh, seq, k, kv="offload", prefetch=pf,
                         trace_queries=tq)
        run(name, dec)
        del dec
        torch.cuda.empty_cache()
    offload = {}
    for sfx in ("", "_trace"):
        ser = results["offload_serial" + sfx]["ms_per_step"]
        pre = results["offload_prefetch" + sfx]["ms_per_step"]
        res = results["resident" + sfx]["ms_per_step"]
        rows = results["offload_prefetch" + sfx]["rows_loaded_per_step"]
        pcie = rows * L * 2 * D * 2
        offload["model_queries" if not sfx else "trace_queries"] = {
            "elastic_reuse": round(1 - rows / (B * G * k), 4),
            "pcie_bytes_per_step": pcie,
            "pcie_gbs_prefetch": round(pcie / (pre * 1e-3) / 1e9, 1),
            # the dense compute hidden under the transfer: prefetch vs serial, relative to the
            # compute time (the resident step); 1 = step time max(compute, transfer)
            "compute_hidden_frac": round(max(0.0, min(1.0, (ser - pre) / min(res, ser - res))), 3)
            if ser > res else None}
    kvb = B * L * G * k * D * 2 * 2
    krb = B * G * (S0 + 1) * D * 2
    ach = (wbytes + kvb + krb) / (ms_res * 1e-3) / 1e9
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
    print(json.dumps({
        "metric": "LLM decode throughput (tokens/s), SpeContext sparse attention", "value":
        results["resident"]["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_res, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights; DESIGN.md §5)",
        "config": {"workload": f"L: llama8b decode, ctx {S0} growing 1/step, batch {B}, k {k}",
                   "l2": "inputs larger than L2 (15 GiB of weights streamed per step)",
                   "variants": results,
                   "offload": dict(offload, what="compute_hidden_frac = (serial - prefetch) / "
                                   "min(resident, serial - resident): the overlap achieved over "
                                   "the overlap possible (P:350)")},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": None,
                     "kernel": "whole resident step: weights + selected KV + retrieval keys"},
        "gpu_launches": results["resident"]["gpu_launches_per_step"] * args.steps,
        "clocks": results["resident"]["clocks"],
        "e2e": {"value": results["resident"]["tokens_per_s"], "unit": "tokens/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4 * B,
                "note": "the generated tokens copied to pinned host memory inside the timed "
                        "region; the next step's input is on the device already"},
    }), flush=True)


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    world = dist_env()[2]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)  # does not return
    if args.dry_run:
        dry_run(args)
        return
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.config is None:
        args.config = "B"
    if args.impl == "reference":
        bench_reference(args)
    elif args.config == "B" and world > 1:
        # the same workload at every N (config B, one request per GPU: weak scaling, no
        # data-path collective), plus config E's 1M-token context sharded over the N ranks
        # (strong scaling, the north star's multi-GPU target) attached to the same line
        sharded = None if args.no_sharded else bench_sharded(args, embedded=True)
        bench_ours(args, attach={"context_sharded_E": sharded})
    elif args.config == "E":
        bench_sharded(args)
    elif args.config == "C":
        bench_grow(args)
    elif args.config == "D":
        bench_offload(args)
    elif args.config == "R":
        bench_frontend(args)
    elif args.config == "M":
        bench_mla(args)
    elif args.config == "O":
        bench_alg2(args)
    elif args.config == "L":
        bench_llm(args)
    else:
        bench_ours(args)
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
