#!/usr/bin/env python
"""bench.py -- VQKV hot-path benchmark on B200 (driver contract).

Headline workload (BASELINE.json configs[1]): 32K-token prefill encode at the
LLaMA3.1-8B KV shape -- 32 layers x 8 KV heads = 256 (layer, head) streams,
D = 128, WindowPolicy{init 4, local 1024} so each stream quantizes its
31,740 middle rows (kv_cache.cpp:76-88) through the key stack (56 x 1024) and
the value stack (16 x 512).  One step = quantize_batch of all 16,250,880 K+V
vectors.  Metric: KV vectors/s VQ-encoded (whole job, all ranks).

Inputs: synthetic, generated with the reference's own generator restated in
the library (synthetic.cpp: rope-rotated mixture keys seed 1000+sid, mixture
values seed 1001+sid); codebooks are the reference's random_stack fixtures
(test_util.hpp, seeds 1 and 2).  Inputs (8.3 GB) exceed L2 (126 MB), so no
flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun, one rank per GPU): every rank encodes its own full
256-stream prefill (weak scaling, no data-path collective); time = max over
ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAYERS, KV_HEADS, D = 32, 8, 128
PREFILL, INIT_LEN, LOCAL_LEN = 32768, 4, 1024
K_SHAPE, V_SHAPE = (56, 1024), (16, 512)
METRIC = "KV vectors/sec VQ-encoded and decode-attn tokens/sec at LLaMA3.1-8B shape"
# L2 -> SM bandwidth measured on this pool's B200s (scripts/micro/l2_gather.cu: bulk copies of 36 KB chunks,
# 2 CTAs per SM, L2-resident source; profiles/r2_decode.md)
L2_PEAK_TBPS = 20.8
UNIT = "KV vectors/s"


def flop_per_vector(n, s):
    return 2 * D * n * s


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=LAYERS * KV_HEADS)
    ap.add_argument("--prefill", type=int, default=PREFILL)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time per baseline sample")
    ap.add_argument("--no-attention", action="store_true")
    ap.add_argument("--attn-context", type=int, default=131072)
    ap.add_argument("--attn-batch", type=int, default=16)
    ap.add_argument("--parity-streams", type=int, default=2,
                    help="full streams of the timed encode output checked against the oracle (0 = skip)")
    ap.add_argument("--parity-pairs", type=int, default=2,
                    help="(sequence, KV head) pairs of the configs[2] attention checked against the oracle")
    return ap.parse_args()


# --------------------------------------------------------------------------- dist
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, local):
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return torch


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- inputs
def gpu_local_cpus(torch, device):
    """Host CPUs on the GPU's NUMA node (sysfs local_cpulist of its PCI function), or None."""
    try:
        p = torch.cuda.get_device_properties(device)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        txt = open(f"/sys/bus/pci/devices/{bdf}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None


def gen_inputs(torch, n_streams, prefill, rank, pinned=True, device=0):
    """Synthetic K/V middle rows [n_streams, middle, D] (host, pinned)."""
    from paper_2603_16435_b200 import _lib

    L = _lib.load()
    middle = prefill - INIT_LEN - LOCAL_LEN
    K = torch.empty((n_streams, middle, D), dtype=torch.float32, pin_memory=pinned)
    V = torch.empty((n_streams, middle, D), dtype=torch.float32, pin_memory=pinned)

    def one(args):
        sid, kind = args
        buf = np.empty((prefill, D), np.float32)
        seed = 1000 + sid + 1_000_000 * rank + (1 if kind == 0 else 0)
        st = L.vqkv_generate_synthetic(1 if kind == 1 else 0, D, prefill, 32, seed, 10000.0, 0.25, 1.0,
                                       buf.ctypes.data)
        assert st == 0
        dst = K if kind == 1 else V
        dst[sid].copy_(torch.from_numpy(buf[INIT_LEN : INIT_LEN + middle]))

    work = [(s, k) for s in range(n_streams) for k in (1, 0)]
    with cf.ThreadPoolExecutor(max_workers=min(64, os.cpu_count() or 8)) as ex:
        list(ex.map(one, work))
    return K, V


def gen_inputs_local(torch, n_streams, prefill, rank, device):
    """gen_inputs with the pinned host buffers allocated and first touched from the CPUs
    of the GPU's NUMA node (H2D from the remote socket runs at a fraction of the link);
    the process affinity is restored afterwards (the CPU baselines use every core)."""
    saved = os.sched_getaffinity(0)
    local = gpu_local_cpus(torch, device)
    try:
        if local:
            os.sched_setaffinity(0, local)
        return gen_inputs(torch, n_streams, prefill, rank, device=device)
    finally:
        if local:
            os.sched_setaffinity(0, saved)


HOST_STACKS = {}  # kind -> (entries, projections): the same bytes the parity checker loads


def make_stacks(device):
    from paper_2603_16435_b200 import _lib, codebook

    L = _lib.load()
    out = []
    for seed, (n, s), kind in ((1, K_SHAPE, 0), (2, V_SHAPE, 1)):
        ent = np.empty((n, s, D), np.float32)
        prj = np.empty((n, D, D), np.float32)
        assert L.vqkv_random_stack(seed, n, s, D, ent.ctypes.data, prj.ctypes.data) == 0
        HOST_STACKS[kind] = (ent, prj)
        out.append(codebook.CodebookStack.from_arrays(list(ent), list(prj), kind, device))
    return out


def oracle_stacks():
    """The checker's copies of the bench stacks (oracle restatement of codebook.cpp, refreshed on
    the host from the same entries and projections the device stacks were built from)."""
    from oracle import oracle as O

    return tuple(O.Stack.from_entries(list(HOST_STACKS[k][0]), list(HOST_STACKS[k][1]), k) for k in (0, 1))


def encode_parity(Kh, Vh, kp, vp, kn, vn, middle, streams):
    """Checker (outside every timed region): the timed encode's output for `streams` full
    streams against the oracle's quantize_batch on the same rows.  Codes bit-exact modulo
    near-ties (tau of SURVEY.md 8c, counted), residual norms bit-exact on every exact row."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    ok, ov = oracle_stacks()
    res = {}
    for name, ost, X, P, N in (("K", ok, Kh, kp, kn), ("V", ov, Vh, vp, vn)):
        tot = dict(rows_checked=0, mismatches=0, near_ties=0, norm_mismatches=0)
        emax = ost.stage_max_norm()
        for sid in streams:
            codes, norms, ins = ost.quantize_rows_instrumented_mt(X[sid].numpy())
            got = ost.unpack(P[sid].cpu().numpy(), middle)
            c = O.classify_codes(got, codes, ins, emax)
            same = (got == codes).all(axis=1)
            gn = N[sid].cpu().numpy()
            tot["norm_mismatches"] += int((gn[same].view(np.uint32) != norms[same].view(np.uint32)).sum())
            for k in ("rows_checked", "mismatches", "near_ties"):
                tot[k] += c[k]
        res[name] = tot
    return {
        "streams": list(streams), "rows_per_stream": middle, "K": res["K"], "V": res["V"],
        "rows_checked": res["K"]["rows_checked"] + res["V"]["rows_checked"],
        "mismatches": res["K"]["mismatches"] + res["V"]["mismatches"],
        "near_ties": res["K"]["near_ties"] + res["V"]["near_ties"],
        "norm_mismatches": res["K"]["norm_mismatches"] + res["V"]["norm_mismatches"],
        "tau": "2^-14 ||r|| max||e|| + 2^-22 max(|s1|,|s2|) at the first differing stage (SURVEY.md 8c)",
        "bar": "codes bit-exact except counted near-ties; residual norms bit-exact (0 ULP)",
        "checker": "oracle/vqkv_oracle.cpp (codebook.cpp:158-237 restated), host threads, outside the timed region",
        "check_s": time.perf_counter() - t0,
    }


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU baseline
def cpu_encode_rate(seconds_target=12.0, threads=None):
    """Oracle (the reference's per-row algorithm restated) on host cores.

    Returns (vectors/s for a 1:1 K:V mix, threads, sample description)."""
    from oracle import oracle as O

    threads = threads or (os.cpu_count() or 1)
    res = {}
    stacks = {"K": O.Rng(1).stack(*K_SHAPE, D, O.KEY), "V": O.Rng(2).stack(*V_SHAPE, D, O.VALUE)}
    desc = []
    for name, kind in (("K", 1), ("V", 0)):
        st = stacks[name]
        # calibrate on a tiny sample, then size the real one
        x = O.generate(kind, D, 4 * threads + INIT_LEN, 32, 1000 + (0 if kind else 1))[INIT_LEN:]
        t0 = time.perf_counter()
        st.quantize_batch_mt(x, threads, 4, threads)
        per_row = (time.perf_counter() - t0) / 4
        rows = max(4, min(4096, int(seconds_target / 2 / max(per_row, 1e-6))))
        x = np.concatenate([O.generate(kind, D, rows + INIT_LEN, 32, 1000 + s + (0 if kind else 1))[INIT_LEN:]
                            for s in range(threads)])
        t0 = time.perf_counter()
        st.quantize_batch_mt(x, threads, rows, threads)
        dt = time.perf_counter() - t0
        res[name] = (threads * rows, dt)
        desc.append(f"{name}: {threads} streams x {rows} rows in {dt:.1f}s")
    (nk, tk), (nv, tv) = res["K"], res["V"]
    rate = 2.0 / (tk / nk + tv / nv)
    return rate, threads, "; ".join(desc) + " (oracle port, one thread per (layer, head) stream, 1:1 K:V mix)"


def cpu_attention_rate(ctx, seconds_target=8.0, threads=None):
    """Oracle attend (attention.cpp:26-69 restated, double-precision online softmax) over
    init | compressed | local segments of a cache of up to `ctx` tokens, one query per host thread.

    Returns (cache tokens/s in the GPU line's B*L/t units, threads, sample description)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    threads = threads or (os.cpu_count() or 1)
    ks, vs = O.Rng(1).stack(*K_SHAPE, D, O.KEY), O.Rng(2).stack(*V_SHAPE, D, O.VALUE)
    n_init, n_local = INIT_LEN, LOCAL_LEN

    def task(n_tok, seed):
        r = np.random.default_rng(seed)
        nc = max(n_tok - n_init - n_local, 0)
        kc = ks.pack(r.integers(0, K_SHAPE[1], (nc, K_SHAPE[0])).astype(np.uint32))
        vc = vs.pack(r.integers(0, V_SHAPE[1], (nc, V_SHAPE[0])).astype(np.uint32))
        f = lambda n: r.standard_normal((n, D)).astype(np.float32)
        a = (ks, vs, f(n_init), f(n_init), kc, vc, nc, f(n_local), f(n_local), f(1)[0])
        t0 = time.perf_counter()
        O.attend_segments(*a)
        return time.perf_counter() - t0

    per_tok = task(4096, 7) / 4096
    n_tok = int(max(2048, min(ctx, seconds_target / max(per_tok, 1e-9))))
    with ThreadPoolExecutor(threads) as ex:
        times = list(ex.map(lambda i: task(n_tok, 1000 + i), range(threads)))  # attend only, per thread
    # the threads ran concurrently: throughput = sum of the per-thread attend rates
    rate = sum(n_tok / t for t in times) / (KV_HEADS * 4)  # token-queries/s -> B*L/t (8 KV heads x G=4 per token)
    return rate, threads, (f"{threads} queries (one per thread, concurrent) x {n_tok} cache tokens, attend "
                           f"{min(times):.1f}-{max(times):.1f}s per thread (code generation untimed); oracle port of "
                           "attend over random codes; normalised to the GPU line's B*L/t units (/ 32 queries per token)")


# --------------------------------------------------------------------------- attention
def bench_attention(torch, Dv, _lib, kst, vst, args, rank, world, local):
    """configs[2]: decode step over a 128K-token compressed cache, batch 16, KV heads
    sharded across ranks (each rank: its KV heads x all 16 sequences, no collective).
    configs[4] (world > 1): one 1M-token sequence split over the ranks, partial
    (o, lse) all-gathered over NCCL and merged by vqkv_lse_combine on every rank.
    Compressed segments hold uniform random codes; raw rows and
    queries are N(0, 1)."""
    from paper_2603_16435_b200 import sharding

    G = 4
    ctx, B = args.attn_context, args.attn_batch
    n_init, n_local = INIT_LEN, LOCAL_LEN
    n_comp = ctx - n_init - n_local
    heads = sharding.kv_head_shard(KV_HEADS, world, rank)
    pairs = B * len(heads)
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    kb, vb = kst.device.payload_bytes(n_comp), vst.device.payload_bytes(n_comp)

    def make(n_pairs, n_comp_, n_init_, n_local_):
        kb_, vb_ = kst.device.payload_bytes(n_comp_), vst.device.payload_bytes(n_comp_)
        # every 10-bit / 9-bit field of random bytes is a valid code (S = 2^bits)
        kc = torch.randint(0, 256, (n_pairs, kb_ + 16), dtype=torch.uint8, device="cuda", generator=gen)[:, :kb_]
        vc = torch.randint(0, 256, (n_pairs, vb_ + 16), dtype=torch.uint8, device="cuda", generator=gen)[:, :vb_]
        kc, vc = kc.contiguous(), vc.contiguous()
        # the key codes as DeviceCacheState keeps them: attention records (transcoded once per
        # flushed row at append time, outside the decode step)
        cap = -(-max(n_comp_, 1) // Dv.GM_ALIGN) * Dv.GM_ALIGN
        kg = Dv.keycodes_to_gm(kst, kc, n_comp_, cap=cap)
        kept["kc"] = kc[: args.parity_pairs].cpu().numpy()  # the checker's copy (CodeMatrix rows)
        del kc
        f = lambda n: (torch.randn(n_pairs, n, D, device="cuda", generator=gen) if n else None)
        return (kg, cap), vc, f(n_init_), f(n_init_), f(n_local_), f(n_local_)

    kept = {}
    (kc, kcap), vc, ik, iv, lk, lv = make(pairs, n_comp, n_init, n_local)
    kc_host = kept["kc"]
    q = torch.randn(pairs, G, D, device="cuda", generator=gen)
    run = lambda: Dv.attend_decode(kst, vst, q, kc, vc, n_comp, ik, iv, lk, lv, kcodes_gm_cap=kcap)
    for _ in range(max(1, args.warmup)):
        run()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    bytes_rank = pairs * (kb + vb) + pairs * (n_init + n_local) * D * 4 * 2 + pairs * G * D * 4 * 2
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6548.8)
    out = {
        "metric": "decode-attn cache tokens/s per layer-step (B*L/t)",
        "config": {"workload": "configs[2]: decode step, 128K-token VQ-compressed cache, batch 16, 8 KV heads "
                               f"sharded over {world} GPU(s), G=4", "context": ctx, "batch": B,
                   "kv_heads_per_gpu": len(heads), "compressed_rows": n_comp, "raw_rows": n_init + n_local,
                   "key_code_layout": "attention records (the cache's only key-code copy, 70 B per token)"},
        "value": B * ctx / (ms / 1e3), "unit": "tokens/s", "ms_per_layer_step": ms,
        "roofline": {"bound": "hbm", "achieved": bytes_rank / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": bytes_rank / (ms / 1e3) / 1e9 / hbm,
                     "algorithmic": "88 B of codes per compressed token-pair + 1 KB per raw row (fp32 K+V)",
                     "note": "on-chip bound: 56 conflict-free 16 B LUT reads per compressed token-pair from shared memory"},
    }
    # the kernel's own bound: shared-memory LUT gathers (main kernel, library profile hooks)
    L = _lib.load()
    L.vqkv_profile_enable(1)
    for nm in (b"attend_lut_build", b"attend", b"attend_combine"):
        L.vqkv_profile_collect(nm, None, None)
    for _ in range(max(2, args.steps)):
        run()
    torch.cuda.synchronize()
    part = {}
    for nm in (b"attend_lut_build", b"attend", b"attend_combine"):
        t_ms, n_l = ctypes.c_double(), ctypes.c_uint64()
        L.vqkv_profile_collect(nm, ctypes.byref(t_ms), ctypes.byref(n_l))
        part[nm.decode()] = t_ms.value / max(1, n_l.value)
    L.vqkv_profile_enable(0)
    smem_peak = 128 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12  # TB/s: 128 B/clk/SM at max clock
    gathers = pairs * n_comp * kst.num_stages() * 16  # one 16 B LUT entry (4 heads) per (token, key stage)
    out["kernel_ms"] = {"lut_gemm": part["attend_lut_build"], "main": part["attend"], "combine": part["attend_combine"]}
    out["onchip"] = {"bound": "shared-memory LUT reads (main kernel)", "algorithmic_bytes": gathers,
                     "achieved": gathers / (part["attend"] / 1e3) / 1e12, "peak": smem_peak, "unit": "TB/s",
                     "frac": gathers / (part["attend"] / 1e3) / 1e12 / smem_peak,
                     "note": "16 B per (compressed token-pair, key stage) at 128 B/clk/SM x 148 SMs x max clock; "
                             "rotated 8-stage rows make every LDS.128 conflict-free (1 wavefront per 8 lanes)"}
    # checker (untimed): the first pairs' outputs against the oracle's attend (attention.cpp:26-69,
    # double-precision online softmax over view_block order), every query head
    o32, _ = run()
    if args.parity_pairs > 0:
        try:
            from concurrent.futures import ThreadPoolExecutor

            from oracle import oracle as O

            t_chk = time.perf_counter()
            ok_, ov_ = oracle_stacks()
            npp = min(args.parity_pairs, pairs)
            host = lambda t: t[:npp].cpu().numpy() if t is not None else None
            hq, hik, hiv, hlk, hlv = (host(t) for t in (q, ik, iv, lk, lv))
            hvc = vc[:npp].cpu().numpy()
            got = o32[:npp].cpu().numpy()

            def one(pg):
                pi, g = divmod(pg, G)
                ref, _ = O.attend_segments(ok_, ov_, hik[pi], hiv[pi], kc_host[pi], hvc[pi], n_comp, hlk[pi], hlv[pi],
                                           hq[pi, g])
                return float(np.abs(got[pi, g] - ref).max() / max(1.0, float(np.abs(ref).max())))

            with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
                devs = list(ex.map(one, range(npp * G)))
            out["parity"] = {
                "pairs_checked": npp, "queries_checked": npp * G, "tokens_per_query": ctx,
                "max_dev": max(devs), "tol": 2.0 ** -7, "pass": bool(max(devs) <= 2.0 ** -7),
                "metric": "max|o - o_ref| / max(1, max|o_ref|) per query (bf16-level bar 2^-7, SURVEY.md 8c)",
                "checker": "oracle attend_segments (attention.cpp:26-69 over kv_cache.cpp:143-189 order), untimed",
                "check_s": time.perf_counter() - t_chk,
            }
        except Exception as e:
            out["parity"] = {"error": repr(e)}
    del kc, vc, ik, iv, lk, lv
    if world > 1:
        # configs[4]: 1M-token single sequence over the ranks, NCCL all-gather + LSE merge
        total = 1 << 20
        sh = sharding.sequence_shards(n_init, total - n_init - n_local, n_local, world)[rank]
        nc = sh.comp[1] - sh.comp[0]
        ni = sh.init[1] - sh.init[0]
        nl = sh.local[1] - sh.local[0]
        (kc, kcap), vc, ik, iv, lk, lv = make(KV_HEADS, nc, ni, nl)
        q1 = torch.randn(KV_HEADS, G, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
        part = lambda: Dv.attend_decode(kst, vst, q1, kc, vc, nc, ik, iv, lk, lv, kcodes_gm_cap=kcap)
        o_l, l_l = part()
        # the exchange step through the library's C-ABI entry (vqkv_lse_allgather_combine) on the
        # process group's own NCCL communicator; torch's all-gather + merge if the pointer is unavailable
        combine_api = "vqkv_lse_allgather_combine"
        try:
            import torch.distributed as dist

            comm = dist.distributed_c10d._get_default_group()._get_backend(torch.device("cuda", local))._comm_ptr()
            combine = lambda: sharding.nccl_gather_and_merge(comm, o_l.reshape(-1, D), l_l.reshape(-1))
            combine()
        except Exception:
            combine_api = "torch.distributed.all_gather_into_tensor + vqkv_lse_combine"
            combine = lambda: sharding.gather_and_merge(o_l, l_l)
            combine()
        torch.cuda.synchronize()
        barrier(world)
        a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a0.record()
        for _ in range(args.steps):
            o_l, l_l = part()
        a1.record()
        for _ in range(args.steps):
            combine()
        a2.record()
        torch.cuda.synchronize()
        kern = max_over_ranks(a0.elapsed_time(a1) / args.steps, world)
        comb = max_over_ranks(a1.elapsed_time(a2) / args.steps, world)
        out["sequence_split_1M"] = {
            "config": f"configs[4]: 1 sequence x 1,048,576 tokens over {world} GPUs, 8 KV heads, G=4",
            "tokens_per_gpu": sh.tokens, "ms_attention_per_layer_step": kern, "ms_nccl_lse_combine": comb,
            "combine_api": combine_api,
            "tokens_per_s": total / ((kern + comb) / 1e3),
        }
    else:
        # configs[4] at N = 1: the same 1M-token sequence on this GPU alone (no split, no collective):
        # the reference point for the N-GPU sequence split above
        total = 1 << 20
        nc = total - n_init - n_local
        (kc, kcap), vc, ik, iv, lk, lv = make(KV_HEADS, nc, n_init, n_local)
        q1 = torch.randn(KV_HEADS, G, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
        one = lambda: Dv.attend_decode(kst, vst, q1, kc, vc, nc, ik, iv, lk, lv, kcodes_gm_cap=kcap)
        for _ in range(max(1, args.warmup)):
            one()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.steps):
            one()
        a1.record()
        torch.cuda.synchronize()
        ms1 = a0.elapsed_time(a1) / args.steps
        b1 = KV_HEADS * (kst.device.payload_bytes(nc) + vst.device.payload_bytes(nc)) + KV_HEADS * (n_init + n_local) * D * 8
        out["sequence_1M_single_gpu"] = {
            "config": "configs[4] at N=1: 1 sequence x 1,048,576 tokens, 8 KV heads, G=4, one GPU (no split)",
            "ms_per_layer_step": ms1, "tokens_per_s": total / (ms1 / 1e3),
            "hbm_gbs": b1 / (ms1 / 1e3) / 1e9, "hbm_frac": b1 / (ms1 / 1e3) / 1e9 / hbm,
        }
        del kc, vc, ik, iv, lk, lv
    return out


# --------------------------------------------------------------------------- arms
def run_reference(args, rank, world):
    if rank != 0:
        return
    rates = []
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up effects; calibration happens inside each step
    cores = 1
    sample = ""
    walls = []
    for _ in range(args.steps):
        t_0 = time.perf_counter()
        r, cores, sample = cpu_encode_rate(seconds_target=max(2.0, args.cpu_seconds / 2))
        walls.append(time.perf_counter() - t_0)
        rates.append(r)
    v = float(np.mean(rates))
    full = 2 * args.streams * (args.prefill - INIT_LEN - LOCAL_LEN)  # K+V vectors of one full step
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.mean(walls)) * 1e3,
        "ms_per_step_basis": "measured wall time of one timed step (a bounded sample of the workload, see "
                             "cpu_baseline.sample); value is that sample's rate",
        "ms_per_full_step_extrapolated": full / v * 1e3,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator, seeds 1000+sid)",
        "config": {"workload": "32K-token prefill encode, LLaMA3.1-8B KV shape (bounded CPU sample)",
                   "streams": args.streams, "rows_per_stream": args.prefill - INIT_LEN - LOCAL_LEN,
                   "key_stack": list(K_SHAPE), "value_stack": list(V_SHAPE), "head_dim": D},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    torch = init_dist(world, local)
    from paper_2603_16435_b200 import _lib
    from paper_2603_16435_b200 import device as Dv

    L = _lib.load()
    kst, vst = make_stacks(local)
    middle = args.prefill - INIT_LEN - LOCAL_LEN
    ns = args.streams
    t_gen = time.perf_counter()
    Kh, Vh = gen_inputs_local(torch, ns, args.prefill, rank, local)
    t_gen = time.perf_counter() - t_gen
    Kd, Vd = Kh.to("cuda", non_blocking=True), Vh.to("cuda", non_blocking=True)
    kp = torch.empty((ns, kst.device.payload_bytes(middle)), dtype=torch.uint8, device="cuda")
    vp = torch.empty((ns, vst.device.payload_bytes(middle)), dtype=torch.uint8, device="cuda")
    kn = torch.empty((ns, middle), dtype=torch.float32, device="cuda")
    vn = torch.empty((ns, middle), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()

    def step():
        Dv.quantize_streams(kst, Kd, payload=kp, norms=kn)
        Dv.quantize_streams(vst, Vd, payload=vp, norms=vn)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    L.vqkv_profile_enable(1)
    L.vqkv_profile_collect(b"encode_tc", None, None)
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
    barrier(world)
    launches = _lib.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    ms_total = max_over_ranks(ms_total, world)
    ms_step = ms_total / args.steps
    enc_ms = ctypes.c_double()
    enc_n = ctypes.c_uint64()
    L.vqkv_profile_collect(b"encode_tc", ctypes.byref(enc_ms), ctypes.byref(enc_n))
    L.vqkv_profile_enable(0)
    vectors_per_rank = 2 * ns * middle
    value = world * vectors_per_rank / (ms_step / 1e3)
    flops_step = ns * middle * (flop_per_vector(*K_SHAPE) + flop_per_vector(*V_SHAPE))
    enc_ms_per_step = enc_ms.value / args.steps
    achieved_tflops = flops_step / (enc_ms_per_step / 1e3) / 1e12
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("bf16_tflops_sustained", 1398.8)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("encode_tc_kernel")

    # ---- parity of the timed output (checker, untimed)
    parity = None
    if rank == 0 and args.parity_streams > 0:
        try:
            sids = sorted({0, ns - 1} if args.parity_streams == 2 else set(range(min(ns, args.parity_streams))))
            parity = encode_parity(Kh, Vh, kp, vp, kn, vn, middle, sids)
        except Exception as e:  # reported, never fatal for the headline line
            parity = {"error": repr(e)}

    # ---- e2e through the public host-buffer API (H2D + encode + D2H each step)
    e2e = None
    if not args.no_e2e:
        kph = torch.empty((ns, kst.device.payload_bytes(middle)), dtype=torch.uint8, pin_memory=True)
        vph = torch.empty((ns, vst.device.payload_bytes(middle)), dtype=torch.uint8, pin_memory=True)
        knh = torch.empty((ns, middle), dtype=torch.float32, pin_memory=True)
        vnh = torch.empty((ns, middle), dtype=torch.float32, pin_memory=True)

        # K and V are independent calls on their own caller streams, and consecutive steps alternate
        # between two such stream pairs (double buffering, as a serving loop would): each call's
        # copy-in is ordered after its own stream's earlier work (stream semantics), so the next
        # step's copies overlap this step's encodes
        e2e_streams = [(torch.cuda.Stream(), torch.cuda.Stream()) for _ in range(2)]
        e2e_i = [0]

        def e2e_fork():
            main = torch.cuda.current_stream()
            for pair in e2e_streams:
                for st in pair:
                    st.wait_stream(main)

        def e2e_join():
            main = torch.cuda.current_stream()
            for pair in e2e_streams:
                for st in pair:
                    main.wait_stream(st)

        def e2e_step():
            sK, sV = e2e_streams[e2e_i[0] & 1]
            e2e_i[0] += 1
            with torch.cuda.stream(sK):
                Dv.quantize_streams_host(kst, Kh, payload_host=kph, norms_host=knh, blocking=False)
            with torch.cuda.stream(sV):
                Dv.quantize_streams_host(vst, Vh, payload_host=vph, norms_host=vnh, blocking=False)

        n_e2e = max(1, min(args.steps, 3))
        # warm-up as many back-to-back steps as are timed: the stream-ordered staging pool grows
        # to its steady-state size (mapping memory) before the timed region
        e2e_fork()
        for _ in range(max(args.warmup, n_e2e)):
            e2e_step()
        e2e_join()
        barrier(world)
        torch.cuda.synchronize()
        # the box's pinned H2D bandwidth (the e2e bound when copies exceed the encode time)
        probe = torch.empty((min(32, ns),) + tuple(Kh.shape[1:]), dtype=torch.float32, device="cuda")
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        probe.copy_(Kh[: probe.shape[0]], non_blocking=True)
        p1.record()
        torch.cuda.synchronize()
        h2d_gbps = probe.numel() * 4 / (p0.elapsed_time(p1) / 1e3) / 1e9
        del probe
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_fork()
        for _ in range(n_e2e):
            e2e_step()
        e2e_join()
        e1.record()
        torch.cuda.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1) / n_e2e, world)
        e2e = {
            "value": world * vectors_per_rank / (e_ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(Kh.numel() * 4 + Vh.numel() * 4),
            "d2h_bytes_per_step": int(kph.numel() + vph.numel() + knh.numel() * 4 + vnh.numel() * 4),
            "ms_per_step": e_ms, "api": "vqkv_quantize_batch_host_async: K and V on their own caller streams, steps alternating between two stream pairs (pinned host buffers), then sync",
            "h2d_gbps_probe": h2d_gbps,
        }

    # ---- decode (K2, reconstruct_block) at the configs[0] shape: 4096 rows of every stream
    decode = None
    try:
        rows_d = min(4096, middle)
        dk = torch.empty((ns, rows_d, D), dtype=torch.float32, device="cuda")
        dv = torch.empty((ns, rows_d, D), dtype=torch.float32, device="cuda")
        dec = lambda: (Dv.reconstruct_streams(kst, kp, middle, 0, rows_d, out=dk),
                       Dv.reconstruct_streams(vst, vp, middle, 0, rows_d, out=dv))
        for _ in range(max(3, args.warmup)):
            dec()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for _ in range(args.steps):
            dec()
        d1.record()
        torch.cuda.synchronize()
        d_ms = max_over_ranks(d0.elapsed_time(d1) / args.steps, world)
        code_bytes = ns * (kst.device.payload_bytes(rows_d) + vst.device.payload_bytes(rows_d))
        out_bytes = 2 * ns * rows_d * D * 4
        gather = ns * rows_d * (K_SHAPE[0] + V_SHAPE[0]) * D * 4
        hbm = (json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.8)
               if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.8)
        decode = {
            "metric": "KV vectors/s reconstructed (reconstruct_block, bit-exact fp32)",
            "config": {"workload": "configs[0] shape: 4096 rows of each of the 256 streams, K 56x1024 + V 16x512"},
            "value": world * 2 * ns * rows_d / (d_ms / 1e3), "unit": "KV vectors/s", "ms_per_step": d_ms,
            "roofline": {"bound": "hbm", "achieved": (code_bytes + out_bytes) / (d_ms / 1e3) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": (code_bytes + out_bytes) / (d_ms / 1e3) / 1e9 / hbm,
                         "algorithmic": "row_bits/8 in + 4*D out per vector",
                         "l2_gather_tbps": gather / (d_ms / 1e3) / 1e12,
                         "l2_peak_tbps_measured": L2_PEAK_TBPS,
                         "l2_frac": gather / (d_ms / 1e3) / 1e12 / L2_PEAK_TBPS,
                         "note": "on-chip bound: one 512 B codebook-row gather from L2 per (vector, stage); "
                                 "l2_frac against the measured L2->SM peak (profiles/r2_decode.md)"},
        }
        if rank == 0 and args.parity_streams > 0:  # checker (untimed): 0 ULP on stream 0's rows
            ok_, ov_ = oracle_stacks()
            ref_k = ok_.reconstruct_block(kp[0].cpu().numpy(), middle, 0, rows_d)
            ref_v = ov_.reconstruct_block(vp[0].cpu().numpy(), middle, 0, rows_d)
            decode["parity"] = {
                "rows_checked": 2 * rows_d,
                "ulp_mismatches": int((dk[0].cpu().numpy().view(np.uint32) != ref_k.view(np.uint32)).sum()
                                      + (dv[0].cpu().numpy().view(np.uint32) != ref_v.view(np.uint32)).sum()),
                "bar": "0 ULP (ordered fp32 sums, codebook.cpp:208-223)",
            }
        del dk, dv
    except Exception as e:  # reported, never fatal for the headline line
        decode = {"error": repr(e)}

    # ---- decode-step attention (configs[2]; configs[4] when world > 1)
    attn = None
    if not args.no_attention:
        try:
            attn = bench_attention(torch, Dv, _lib, kst, vst, args, rank, world, local)
        except Exception as e:  # reported, never fatal for the headline line
            attn = {"error": repr(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r, cores, sample = cpu_encode_rate(args.cpu_seconds)
            cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {e}"}
        if attn is not None and "error" not in attn:
            try:
                r, cores, sample = cpu_attention_rate(args.attn_context, seconds_target=args.cpu_seconds / 2)
                attn["cpu_baseline"] = {"value": r, "unit": "tokens/s", "cores": cores, "kind": "port",
                                        "sample": sample}
            except Exception as e:
                attn["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "port",
                                        "sample": f"failed: {e}"}

    if rank == 0:
        counters = Dv.encode_counters(kst)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16 MMA / f32 exact (indices bit-exact)",
            "data": "synthetic (reference generator: rope-rotated mixture keys, mixture values; random_stack codebooks)",
            "config": {
                "workload": "32K-token prefill encode (configs[1]), LLaMA3.1-8B KV shape",
                "streams_per_gpu": ns, "layers": LAYERS, "kv_heads": KV_HEADS, "head_dim": D,
                "rows_per_stream": middle, "key_stack": list(K_SHAPE), "value_stack": list(V_SHAPE),
                "kv_vectors_per_gpu": vectors_per_rank, "l2": "inputs (8.3 GB) larger than L2, no flush",
                "parallelism": f"dp{world} (independent prefills per GPU)",
            },
            "roofline": {
                "bound": "tensor", "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tflops / peak, "traffic": traffic,
                "kernel": "encode_tc_kernel", "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                "algorithmic": "2*D*N*S flop per vector (K 14,680,064; V 2,097,152)",
                "kernel_ms_per_step": enc_ms_per_step, "kernel_launches": int(enc_n.value),
            },
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "decode": decode,
            "decode_attention": attn,
            "ambiguous_row_stage_frac_K": counters["ambiguous"] / max(1, counters["row_stages"]),
            "input_gen_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
