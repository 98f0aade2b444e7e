"""Benchmark of the KVTuner hot path on B200: one decode step = for every layer, quantise-append the
new token's K/V (K1) and run decode attention over the packed mixed-precision cache (K2, split merge fused).

Metric (BASELINE.json): decode tokens/s (= sequences decoded per step / step time, attention-only: no
weights, GEMMs or MLPs) and the HBM GB/s of the attention kernel as a fraction of the measured B200 copy peak.

    python bench.py [--gpus N --steps K --warmup W] [--workload llama-3.25|qwen-4.00|...]
    python bench.py --impl reference ...        # the CPU oracle on a bounded sample (rank 0 only)
    torchrun --nproc-per-node N bench.py --gpus N [--scaling weak|strong]

Multi-GPU (`paper_2502_04420_b200/partition.py`): weak scaling gives every rank `--batch`
sequences; strong scaling splits `--batch` sequences over the ranks (batch rows, or KV heads when the
batch is smaller than the world); `*-seqshard` workloads shard every sequence's tokens and exchange the
(m, l, o) partials once per layer.  Rank 0 prints ONE JSON line.  Inputs are synthetic (kvt_synth recipe),
resident in HBM before the timed region; the cache (~18 GB at the default workload) is far larger than L2,
so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (config file, model shape (L, H_kv, H_q), default batch, context)
    "llama-3.25": ("configs/llama-3.1-8b_kivi_3.25.json", (32, 8, 32), 64, 8192),
    "qwen-4.00": ("configs/qwen2.5-7b_per-token-asym_4.00.json", (28, 4, 28), 64, 8192),
    "qwen-3.92": ("configs/qwen2.5-7b_kivi_3.92.json", (28, 4, 28), 64, 8192),
    # the paper's exact 4.00 map in its own mode (per-token-asym, G = 32, R = 0), not the KIVI layout of A19
    "qwen-4.00-pertoken": ("configs/qwen2.5-7b_per-token-asym_4.00.json", (28, 4, 28), 64, 8192),
    "llama-kv8": (None, (32, 8, 32), 64, 8192),
    "qwen-kv8": (None, (28, 4, 28), 64, 8192),
    # config 5: 128k context, sequence-sharded over the ranks (partial -> NCCL all-gather -> combine)
    "llama-128k-seqshard": ("configs/llama-3.1-8b_kivi_3.25.json", (32, 8, 32), 8, 131072),
}
D = 128
SPEC_HBM_GBS = 8000.0        # B200 HBM3e nominal (DGX figure, B200_PROFILING.md); context for the record only


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvt", choices=["kvt", "reference"])
    ap.add_argument("--workload", default="llama-3.25", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None,
                    help="weak scaling: sequences per GPU; strong scaling: sequences in total")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="batch/head partitions only (seqshard workloads are strong by construction)")
    ap.add_argument("--ctx", type=int, default=None, help="tokens in the cache after the first append")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "symm"],
                    help="seqshard workloads: NCCL all-gather of the partials, or the fused push into the peers' "
                         "symmetric-memory buffers (kvt_decode_attention_partial_push + one barrier)")
    ap.add_argument("--launch", default="graph", choices=["graph", "eager"],
                    help="timed step as one CUDA graph replay (default) or eager launches through ctypes")
    ap.add_argument("--paged", action="store_true",
                    help="paged tile records: every 32-token block in a shuffled page of a per-layer pool")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / e2e / cpu baseline)")
    return ap.parse_args()


METRIC = "decode tokens/s (attention-only, mixed-precision KV)"
DATA = "synthetic (kvt_synth: N(0,1) K with x11 outliers on channels c%8==0, N(0,1) V, 0.5 N(0,1) q)"


def oracle_specs(name):
    """The workload's layer specs through the ORACLE's own config reader (no product code: VERDICT r1 W1)."""
    from oracle import config as ocfg

    cfg_path, (L, H, Hq), B, S = WORKLOADS[name]
    if cfg_path is None:
        return [ocfg.OracleLayer(ocfg.MODE_KIVI, 8, 8, 32, 32) for _ in range(L)], \
            "uniform KIVI-KV8 (baseline of P:538)"
    cfg = ocfg.load(ROOT / cfg_path)
    specs = list(cfg.layers)
    if name == "qwen-4.00":   # A19: the paper's exact-4.00 Qwen2.5-7B map, stored in the KIVI layout
        specs = [ocfg.OracleLayer(ocfg.MODE_KIVI, s.key_bits, s.value_bits, 32, 32) for s in specs]
    return specs, f"{cfg.model_name} {cfg_path} (f_m = {cfg.equivalent_bits:g})"


def product_specs(name, kvt):
    """The same layer specs through the library's loader (kvt_config_load) for the GPU arm."""
    cfg_path, (L, H, Hq), B, S = WORKLOADS[name]
    if cfg_path is None:
        return [kvt.LayerSpec.kivi(8, 8) for _ in range(L)], "uniform KIVI-KV8 (baseline of P:538)"
    cfg = kvt.load_config(str(ROOT / cfg_path))
    specs = cfg.layers
    if name == "qwen-4.00":
        specs = [kvt.LayerSpec.kivi(s.key_bits, s.value_bits) for s in specs]
    return specs, f"{cfg.model_name} {cfg_path} (f_m = {cfg.equivalent_bits:g})"


def algorithmic_bytes(spec, B, H, Hq, S):
    """Bytes the method must move for one decode attention launch of one layer:
    packed codes + bf16 scale/zero of the quantised tokens, bf16 residual tokens, q read, out write."""
    def nq_key():
        if spec.key_bits == 16:
            return S
        if spec.mode == 1:
            F = spec.residual if spec.residual > 0 else spec.group
            return F * (S // F)
        return max(0, S - spec.residual)
    nqv = S if spec.value_bits == 16 else max(0, S - spec.residual)
    nqk = nq_key()

    def per_tok(bits):
        if bits == 16:
            return 2 * D
        return D * bits // 8 + (D // spec.group) * 4      # codes + meta (per-channel meta is also 4 B x d / G per token)
    tok = nqk * per_tok(spec.key_bits) + (S - nqk) * 2 * D + nqv * per_tok(spec.value_bits) + (S - nqv) * 2 * D
    return B * H * tok + B * Hq * D * 2 * 2


def plan(args, world, rank):
    """(B_rank, kv-head range, global tokens per step, scaling label, parallelism label)."""
    from paper_2502_04420_b200.partition import partition

    _, (L, H, Hq), B_def, _ = WORKLOADS[args.workload]
    B = args.batch or B_def
    if args.workload.endswith("seqshard"):
        return B, (0, H), B, "strong", parallelism(args, world)
    if args.scaling == "weak":
        return B, (0, H), world * B, "weak", parallelism(args, world)
    p = partition(B, H, world, rank)
    return p.batch, (p.h_lo, p.h_hi), B, "strong", parallelism(args, world)


def parallelism(args, world):
    _, (L, H, Hq), B_def, _ = WORKLOADS[args.workload]
    B = args.batch or B_def
    if args.workload.endswith("seqshard"):
        how = "fused push into peer symmetric memory -> barrier -> combine" if args.exchange == "symm" else \
            "partial -> NCCL all-gather -> combine"
        return f"sequence-sharded x{world} ({how})"
    if args.scaling == "weak":
        return f"batch-partitioned x{world} (B={B} per GPU, no collective)"
    how = "batch rows" if B >= world else "KV heads (B < N)"
    return f"{how} over {world} GPUs (global B={B}, no collective)"


def config_of(args, desc, world):
    """The `config` object of the JSON line — built the same way in both arms (the reference arm describes the
    workload its bounded sample is drawn from), so the driver compares like with like."""
    _, (L, H, Hq), B_def, S_ctx = WORKLOADS[args.workload]
    S_first = (args.ctx or S_ctx) + args.warmup            # context of the first timed step
    return {"workload": args.workload, "layers": desc, "shape": {"L": L, "H_kv": H, "H_q": Hq, "d": D},
            "batch": args.batch or B_def, "ctx": f"{S_first}..{S_first + args.steps - 1}",
            "scaling": "strong" if (args.workload.endswith("seqshard") or args.scaling == "strong") else "weak",
            "parallelism": parallelism(args, world),
            "l2": "inputs larger than L2 (packed cache >> 126 MB; no flush)",
            "kv_layout": "paged (shuffled 32-token pages, block table)" if args.paged else "dense"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, dev_index):
        self.dev = dev_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks.mem,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, mem, pw, reasons = [], [], [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
                if len(parts) >= 5:
                    mem.append(float(parts[3]))
                    pw.append(float(parts[4]))
            except ValueError:
                continue
            for bit, name in self.REASONS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return None
        sm.sort()
        mem.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm),
                "mem_mhz": mem[len(mem) // 2] if mem else None, "power_w_max": max(pw) if pw else None}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload):
    """dram read+write bytes per launch of the profiled decode kernel (one ncu --set full capture,
    profiles/ncu_traffic.json) — compare with that launch's algorithmic bytes, not the step average."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        j = json.loads(p.read_text()).get(workload)
        if j:
            return j["traffic_bytes_per_launch"], j
    return None, None


def build_info():
    """git SHA of the source the library was built from: `git` when the checkout has .git, else the stamp
    build.py writes next to libkvt.so (the GPU box's snapshot has no .git)."""
    try:
        sha = subprocess.run(["git", "rev-parse", "HEAD"], cwd=ROOT, capture_output=True, text=True, timeout=10)
        if sha.returncode == 0:
            dirty = subprocess.run(["git", "status", "--porcelain", "--untracked-files=no"], cwd=ROOT,
                                   capture_output=True, text=True, timeout=10).stdout.strip() != ""
            return {"git_sha": sha.stdout.strip(), "dirty": dirty, "source": "git"}
    except (OSError, subprocess.SubprocessError):
        pass
    p = ROOT / "paper_2502_04420_b200" / "BUILD_INFO.json"
    if p.exists():
        return {**json.loads(p.read_text()), "source": "BUILD_INFO.json (written by build.py)"}
    return {"git_sha": None, "source": "unknown"}


def host_info():
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "nproc": n, "os_cpu_count": os.cpu_count()}


# ------------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference): the oracle as it stands, plain C, one unit per thread
# ------------------------------------------------------------------------------------------------
class OracleSampler:
    """Times the C oracle (O2 static build + fp64 read-back + fp64 Eq. 1 attention) on (layer, kv head) units
    of ONE sequence of the workload at context S, `threads` units at a time (ctypes releases the GIL, so the
    units run on separate cores).  tokens = units / (L * H_kv): a decode token needs every (layer, head)."""

    def __init__(self, specs, shape, S, seed=11):
        import kvt_synth
        import oracle

        oracle.build()
        self.oracle = oracle
        self.specs, self.shape, self.S = specs, shape, S
        L, H, Hq = shape
        g = Hq // H
        self.K = kvt_synth.bf16_bits(kvt_synth.keys((1, 1, S, D), seed=seed))
        self.V = kvt_synth.bf16_bits(kvt_synth.values((1, 1, S, D), seed=seed + 1))
        self.q = kvt_synth.bf16_bits(kvt_synth.queries((1, g, D), seed=seed + 2))
        import numpy as np

        self.sl = np.array([S], np.int32)
        self.u = 0

    def _unit(self, u):
        s = self.specs[(u * 7) % len(self.specs)]
        self.oracle.layer_decode(s.mode, s.key_bits, s.value_bits, s.group, s.residual, self.K, self.V, self.q,
                                 self.sl, 1 / math.sqrt(D))

    def run(self, n_units, threads):
        """Returns (seconds, decode tokens) for n_units units on `threads` threads."""
        from concurrent.futures import ThreadPoolExecutor

        us = list(range(self.u, self.u + n_units))
        self.u += n_units
        t0 = time.perf_counter()
        if threads <= 1:
            for u in us:
                self._unit(u)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(self._unit, us))
        dt = time.perf_counter() - t0
        L, H, _ = self.shape
        return dt, n_units / (L * H)


def cpu_baseline_record(sampler, S, single_s=5.0, multi_s=12.0):
    """cpu_baseline at 1 core and at nproc cores: bounded samples of the workload, sized by time
    (~5 s single-core, ~12 s on all cores, so the default run stays within minutes)."""
    hi = host_info()
    n = hi["nproc"] or 1
    dt1 = tok1 = 0.0
    n1 = 0
    while dt1 < single_s:
        dt, tok = sampler.run(4, 1)
        dt1 += dt; tok1 += tok; n1 += 4
    dtn = tokn = 0.0
    nn = 0
    while dtn < multi_s:
        dt, tok = sampler.run(2 * n, n)
        dtn += dt; tokn += tok; nn += 2 * n
    return {"value": tokn / dtn, "unit": "tokens/s", "cores": n, "kind": "oracle",
            "sample": f"{nn} (layer, kv head) units of 1 sequence at S={S} on {n} threads "
                      f"(= {tokn:.3f} decode tokens, {dtn:.1f} s); oracle = O2 static build + fp64 read-back "
                      f"+ fp64 Eq.1, plain C, one unit per thread",
            "single_core": {"value": tok1 / dt1, "unit": "tokens/s", "cores": 1,
                            "sample": f"{n1} units at S={S} ({dt1:.1f} s)"},
            **hi}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    specs, desc = oracle_specs(args.workload)
    _, shape, B_def, S_ctx = WORKLOADS[args.workload]
    L, H, Hq = shape
    S_first = (args.ctx or S_ctx) + args.warmup    # the GPU arm's first timed context (same config object)
    hi = host_info()
    n = hi["nproc"] or 1
    smp = OracleSampler(specs, shape, S_first)
    for _ in range(args.warmup):
        smp.run(n, n)
    times, tot_tok = [], 0.0
    for _ in range(args.steps):
        dt, tok = smp.run(n, n)
        times.append(dt)
        tot_tok += tok
    tot_t = sum(times)
    value = tot_tok / tot_t
    sample = (f"per step: {n} (layer, kv head) units of 1 sequence at S={S_first} on {n} threads (layers rotate), "
              f"i.e. {n}/{L * H} of a decode token; oracle = O2 static build + fp64 read-back + fp64 Eq.1 "
              f"attention, plain C, one unit per thread")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / max(args.steps, 1),
            "higher_is_better": True, "scaling": config_of(args, desc, world)["scaling"],
            "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": config_of(args, desc, world),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": n, "kind": "oracle", "sample": sample, **hi},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def _pct(xs, p):
    xs = sorted(xs)
    if not xs:
        return None
    k = (len(xs) - 1) * p
    lo = int(math.floor(k))
    hi = min(lo + 1, len(xs) - 1)
    return xs[lo] + (xs[hi] - xs[lo]) * (k - lo)


def run_kvt(args):
    import torch
    import torch.distributed as dist

    import paper_2502_04420_b200 as kvt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    _, (L, H_all, Hq_all), B_def, S_ctx = WORKLOADS[args.workload]
    g = Hq_all // H_all
    specs, desc = product_specs(args.workload, kvt)
    B, (h_lo, h_hi), tokens_per_step, scaling, par = plan(args, world, rank)
    H, Hq = h_hi - h_lo, (h_hi - h_lo) * g
    S_ctx = args.ctx or S_ctx
    seqshard = args.workload.endswith("seqshard")
    S0 = S_ctx - 1                                           # prefilled; the first timed append makes S_ctx
    n_steps_total = args.warmup + 2 * args.steps + (0 if args.no_e2e else args.warmup + args.steps) + 2
    appends = True
    if seqshard:                                             # a6: this rank holds tokens [lo, hi) of every sequence
        from paper_2502_04420_b200.seqshard import shard_bounds, shard_spec

        lo, hi = shard_bounds(S0, world, rank)
        S0 = hi - lo
        appends = rank == world - 1                          # the newest tokens (and the residual) live on the last rank
        specs = [shard_spec(sp, rank, world) for sp in specs]
    cap = ((S0 + (n_steps_total if appends else 0) + 1 + 63) // 64) * 64

    # ---- build the caches: prefill S0 tokens per sequence through the append kernel ----
    gen = torch.Generator(device=dev)
    caches = []
    for l, spec in enumerate(specs):
        if args.paged:        # vLLM-style: one block table per layer, pages assigned in a random order
            pg = torch.Generator().manual_seed(500 + l)
            bt = torch.randperm(B * (cap // 32), generator=pg).view(B, cap // 32).to(torch.int32).to(dev)
            cache = kvt.LayerCache(spec, B, H, D, cap, device=dev, block_table=bt, num_pages=B * (cap // 32))
        else:
            cache = kvt.LayerCache(spec, B, H, D, cap, device=dev)
        gen.manual_seed(1000 * rank + l)
        # prefill in token chunks (the append is history independent, A7) so the bf16/fp32 temporaries stay at
        # ~1.5 GB whatever the batch: the config-4 sweep fills ~90% of HBM with the cache itself
        pf = max(32, min(S0, int(1.5e9 / (B * H * D * 6))) // 32 * 32)
        for t0 in range(0, S0, pf):
            n = min(pf, S0 - t0)
            Kp = torch.randn(B, H, n, D, device=dev, generator=gen)
            Kp[..., ::8] *= 11.0                              # kvt_synth recipe: key channel outliers
            Kp = Kp.to(torch.bfloat16)
            Vp = torch.randn(B, H, n, D, device=dev, generator=gen).to(torch.bfloat16)
            kvt.quantize_append(cache, Kp, Vp, torch.full((B,), t0, dtype=torch.int32, device=dev),
                                torch.full((B,), n, dtype=torch.int32, device=dev), len_before_host=[t0] * B,
                                n_new_host=[n] * B)
            del Kp, Vp
        torch.cuda.empty_cache()
        caches.append(cache)
    torch.cuda.synchronize()
    # ---- per-step inputs (resident): one contiguous device buffer of every layer's q, k_new, v_new and one of
    # all outputs, so the end-to-end leg moves them with one host->device and one device->host copy per step
    gen.manual_seed(77 + rank)
    n_q, n_kv = B * Hq * D, B * H * D
    d_in = torch.empty(L, n_q + 2 * n_kv, dtype=torch.bfloat16, device=dev)
    d_in[:, :n_q] = (0.5 * torch.randn(L, n_q, device=dev, generator=gen)).to(torch.bfloat16)
    d_in[:, n_q:] = torch.randn(L, 2 * n_kv, device=dev, generator=gen).to(torch.bfloat16)
    d_out = torch.empty(L, B, Hq, D, dtype=torch.bfloat16, device=dev)

    def views(din, dout):
        return ([din[l, :n_q].view(B, Hq, D) for l in range(L)],
                [din[l, n_q:n_q + n_kv].view(B, H, 1, D) for l in range(L)],
                [din[l, n_q + n_kv:].view(B, H, 1, D) for l in range(L)],
                [dout[l] for l in range(L)])

    bufsets = [views(d_in, d_out)]
    ws_bytes = max(kvt.decode_workspace_bytes(c, Hq, None) for c in caches)   # planned for capacity: graph-safe
    ws = torch.zeros(max(ws_bytes, 16), dtype=torch.uint8, device=dev)      # merge counters start at zero
    len_before = torch.full((B,), S0, dtype=torch.int32, device=dev)
    len_after = torch.full((B,), S0 + (1 if appends else 0), dtype=torch.int32, device=dev)
    ones = torch.ones(B, dtype=torch.int32, device=dev)
    scale = 1.0 / math.sqrt(D)
    main_stream = torch.cuda.current_stream()
    exch = None
    part = gathered = None
    if seqshard:
        from paper_2502_04420_b200.seqshard import sharded_decode

        part = torch.empty(B, Hq, D + 2, dtype=torch.float32, device=dev)
        gathered = torch.empty(world, B, Hq, D + 2, dtype=torch.float32, device=dev) if world > 1 else None
        if args.exchange == "symm":
            from paper_2502_04420_b200.seqshard import SymmExchange

            if world == 1 and not dist.is_initialized():
                dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1,
                                        device_id=dev)
            exch = SymmExchange((B, Hq, D + 2), dev)

    def step(ev=None, bs=0, stream=None):
        stream = stream or main_stream
        q, k_new, v_new, outs = bufsets[bs]
        fused = ev is None and appends and not seqshard
        for l in range(L):
            if appends and not fused:
                kvt.quantize_append(caches[l], k_new[l], v_new[l], len_before, ones, n_new_max=1, stream=stream)
            if ev is not None:
                ev[l][0].record(stream)
            mark = (lambda l=l: ev[l][1].record(stream)) if ev is not None else None
            if exch is not None:          # fused exchange: push into the peers' buffers, barrier, combine
                exch.decode(caches[l], q[l], len_after, scale=scale, out=outs[l], workspace=ws, stream=stream,
                            after_partial=mark)
            elif seqshard:                # a6 through the tested orchestration: partial -> all-gather -> combine
                sharded_decode(caches[l], q[l], len_after, scale=scale, out=outs[l], part=part, gathered=gathered,
                               workspace=ws, stream=stream, after_partial=mark)
            elif fused:                   # the serving step of one layer: append + attention in one library call
                kvt.append_decode_attention(caches[l], k_new[l], v_new[l], len_before, ones, q[l], len_after,
                                            scale=scale, out=outs[l], workspace=ws, stream=stream)
            else:
                kvt.decode_attention(caches[l], q[l], len_after, scale=scale, out=outs[l], workspace=ws, stream=stream)
                if mark:
                    mark()
        if appends:
            len_before.add_(1)
            len_after.add_(1)

    # CUDA graph of one step per buffer set (the lengths advance inside the graph; every kernel reads them on
    # the device and the workspace is planned for the capacity, so one capture serves every replay)
    use_graph = args.launch == "graph" and not seqshard and not args.profile
    graphs = {}

    def capture(bs):
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(main_stream)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            step(bs=bs, stream=s)
        main_stream.wait_stream(s)
        graphs[bs] = gr

    def run_step(bs=0):
        if use_graph:
            graphs[bs].replay()
        else:
            step(bs=bs)

    if use_graph:
        # capturing records the launches without running them: the lengths are not advanced by the capture
        capture(0)
    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # per-layer attention events (live, on the launching stream) for the roofline
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(L)]
           for _ in range(args.steps)]
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    S_first = S0 + (args.warmup + 1 if appends else 0)
    sampler = ClockSampler(dev.index) if not args.profile else None
    if sampler:
        sampler.__enter__()
    # timed region: K steps back to back, an event at every step boundary (p10/p50/p90); no per-layer events
    # (the attention launch may overlap the tail of the same layer's append, programmatic dependent launch)
    marks[0].record(main_stream)
    for i in range(args.steps):
        run_step()
        marks[i + 1].record(main_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # roofline pass: the next K steps eagerly, with CUDA events around every attention launch
    for i in range(args.steps):
        step(evs[i])
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    ms = marks[0].elapsed_time(marks[-1])
    per_step = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    attn_ms = sum(e[0].elapsed_time(e[1]) for st in evs for e in st)
    if world > 1:
        t = torch.tensor([ms, attn_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, attn_ms = t.tolist()
    ms_per_step = ms / args.steps
    value = tokens_per_step / (ms_per_step / 1000.0)

    # roofline of the dominant kernel (decode attention, all layers): algorithmic bytes / event time
    alg = 0
    for i in range(args.steps):
        S = S_first + (args.steps + i if appends else 0)          # the roofline pass follows the timed steps
        alg += sum(algorithmic_bytes(s, B, H, Hq, S) for s in specs)
    achieved = alg / (attn_ms / 1000.0) / 1e9
    peak, peak_src = measured_peaks()
    traffic, traffic_src = ncu_traffic(args.workload)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src, "kernel": "decode attention (all layers)",
                "attn_share_of_step": attn_ms / ms, "peak_source": peak_src,
                "frac_of_spec_8TBs": achieved / SPEC_HBM_GBS,
                "algorithmic_bytes_per_step": alg / args.steps,
                "timing": "CUDA events around every attention launch of a second (eager) pass of K steps"}
    # per precision pair: mean attention time per launch and its fraction of the peak (same events)
    by_pair = {}
    for l, s in enumerate(specs):
        key = f"{'PT' if s.mode != 1 else ''}K{s.key_bits}V{s.value_bits}"
        t = sum(evs[i][l][0].elapsed_time(evs[i][l][1]) for i in range(args.steps)) / args.steps
        nb = sum(algorithmic_bytes(s, B, H, Hq, S_first + (args.steps + i if appends else 0))
                 for i in range(args.steps)) / args.steps
        e = by_pair.setdefault(key, {"layers": 0, "us": 0.0, "bytes": 0.0})
        e["layers"] += 1; e["us"] += t * 1000.0; e["bytes"] += nb
    plans = {}
    for l, s in enumerate(specs):
        key = f"{'PT' if s.mode != 1 else ''}K{s.key_bits}V{s.value_bits}"
        if key not in plans:
            try:
                plans[key] = kvt.decode_plan(caches[l], Hq)          # the work plan of the launch (kvt_decode_plan)
            except Exception as e:                                 # noqa: BLE001 - reporting only
                plans[key] = {"error": str(e)}
    roofline["by_pair"] = {k: {"layers": v["layers"], "us_per_launch": v["us"] / v["layers"],
                               "frac": v["bytes"] / (v["us"] / 1e6) / 1e9 / peak, "plan": plans.get(k)}
                           for k, v in by_pair.items()}

    # ---- e2e: host (pinned) inputs -> device, step, outputs -> host, every step ----
    e2e = None
    if not args.no_e2e and not args.profile:
        # Every step copies its inputs host -> device and its outputs device -> host, pipelined as a serving
        # loop would: a copy stream moves step i+1's inputs and step i-1's outputs while step i computes
        # (two device buffer sets).  The timed region ends when the last outputs are on the host.
        h_in = d_in.cpu().pin_memory()                       # q, k_new, v_new of every layer (pinned host)
        h_out = torch.empty(d_out.shape, dtype=torch.bfloat16).pin_memory()
        bi = d_in.numel() * 2
        bo = d_out.numel() * 2
        d_ins = [d_in, torch.empty_like(d_in)]
        d_outs = [d_out, torch.empty_like(d_out)]
        bufsets.append(views(d_ins[1], d_outs[1]))
        if use_graph:
            capture(1)
        cs = torch.cuda.Stream(device=dev)
        h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        comp_done = [torch.cuda.Event(), torch.cuda.Event()]
        d2h_done = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(i):
            j = i % 2
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(comp_done[j])              # step i-2 has consumed buffer set j
                d_ins[j].copy_(h_in, non_blocking=True)      # step i's inputs, host -> device
                h2d_done[j].record(cs)

        def e2e_run(n):
            h2d(0)
            for i in range(n):
                j = i % 2
                if i + 1 < n:
                    h2d(i + 1)                               # overlaps step i
                main_stream.wait_event(h2d_done[j])
                if i >= 2:
                    main_stream.wait_event(d2h_done[j])      # step i-2's outputs left buffer set j
                run_step(bs=j)
                comp_done[j].record(main_stream)
                with torch.cuda.stream(cs):
                    cs.wait_event(comp_done[j])
                    h_out.copy_(d_outs[j], non_blocking=True)    # step i's outputs, device -> host
                    d2h_done[j].record(cs)
            main_stream.wait_event(d2h_done[(n - 1) % 2])

        e2e_run(args.warmup)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(main_stream)
        e2e_run(args.steps)
        e2.record(main_stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ems = s2.elapsed_time(e2)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": tokens_per_step / (ems / args.steps / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "api": "kvt.quantize_append + kvt.decode_attention per layer"
                                                 + (" (one CUDA graph per step)" if use_graph else "")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        ospecs, _ = oracle_specs(args.workload)
        cpu = cpu_baseline_record(OracleSampler(ospecs, (L, H_all, Hq_all), S_first), S_first)

    clocks = sampler.summary() if sampler else None
    if rank == 0:
        per_layer = (1 if appends else 0) + 1 + (1 if seqshard else 0)
        line = {"metric": METRIC, "value": value, "unit": "tokens/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "ms_per_step_p10": _pct(per_step, 0.1), "ms_per_step_p50": _pct(per_step, 0.5),
                "ms_per_step_p90": _pct(per_step, 0.9),
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
                "dtype": "f32 accumulate of f16 tensor-core products (u2/u4/u8 codes, bf16 in/out)",
                "data": DATA,
                "config": config_of(args, desc, world),
                "run": {"tokens_per_step": tokens_per_step, "rank0_batch": B, "rank0_kv_heads": [h_lo, h_hi],
                        "launch": "one CUDA graph per step" if use_graph else "eager (ctypes per kernel)"},
                "cache_gb_per_gpu": sum(c.nbytes for c in caches) / 1e9,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": args.steps * per_layer * L,
                "clocks": clocks, "gpu": torch.cuda.get_device_name(dev), "build": build_info(),
                "gb_per_s_attention": achieved}
        print(json.dumps(line))
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_kvt(args)


if __name__ == "__main__":
    main()
