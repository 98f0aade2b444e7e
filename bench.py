"""Benchmark of the KVTuner hot path on B200: one decode step = for every layer, quantise-append the
new token's K/V (K1) and run decode attention over the packed mixed-precision cache (K2 + K3).

Metric (BASELINE.json): decode tokens/s (= batch / step time, attention-only: no weights, GEMMs or
MLPs) and the HBM GB/s of the attention kernel as a fraction of the measured B200 copy peak.

    python bench.py [--gpus N --steps K --warmup W] [--workload llama-3.25|qwen-4.00|llama-kv8|qwen-kv8]
    python bench.py --impl reference ...        # the CPU oracle on a bounded sample (rank 0 only)
    torchrun --nproc-per-node N bench.py --gpus N ...   (weak scaling: B sequences per GPU)

Rank 0 prints ONE JSON line.  Inputs are synthetic (kvt_synth recipe), resident in HBM before the
timed region; the cache (~18 GB at the default workload) is far larger than L2, so no L2 flush is
needed between steps.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvt", choices=["kvt", "reference"])
    ap.add_argument("--workload", default="llama-3.25", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU (weak scaling)")
    ap.add_argument("--ctx", type=int, default=None, help="tokens in the cache after the first append")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "symm"],
                    help="seqshard workloads: NCCL all-gather of the partials, or the fused push into the peers' "
                         "symmetric-memory buffers (kvt_decode_attention_partial_push + one barrier)")
    ap.add_argument("--paged", action="store_true",
                    help="paged tile records: every 32-token block in a shuffled page of a per-layer pool")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / e2e / cpu baseline)")
    return ap.parse_args()


def layer_specs(name, kvt):
    cfg_path, (L, H, Hq), B, S = WORKLOADS[name]
    name = name.replace("-128k-seqshard", "-3.25")
    if cfg_path is None:
        return [kvt.LayerSpec.kivi(8, 8) for _ in range(L)], "uniform KIVI-KV8 (baseline of P:538)"
    cfg = kvt.load_config(str(ROOT / cfg_path))
    specs = cfg.layers
    if name == "qwen-4.00":   # A19: the paper's exact-4.00 Qwen2.5-7B map, stored in the KIVI layout
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

    def per_tok(bits, per_channel):
        if bits == 16:
            return 2 * D
        return D * bits // 8 + (D // spec.group) * 4      # codes + meta (per-channel meta is also 4 B x d / G per token)
    tok = nqk * per_tok(spec.key_bits, spec.mode == 1) + (S - nqk) * 2 * D \
        + nqv * per_tok(spec.value_bits, False) + (S - nqv) * 2 * D
    return B * H * tok + B * Hq * D * 2 * 2


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
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
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
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for bit, name in self.REASONS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


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


# ------------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference): the oracle as it stands, single-threaded C
# ------------------------------------------------------------------------------------------------
def oracle_sample(specs, shape, S, n_units, seed=11):
    """Time the oracle on `n_units` (layer, kv head) units of ONE sequence of the workload (layers
    rotate).  Returns (seconds, tokens) where tokens = units / (L * H_kv) decode tokens."""
    import numpy as np

    import kvt_synth
    import oracle

    oracle.build()
    L, H, Hq = shape
    g = Hq // H
    K = kvt_synth.bf16_bits(kvt_synth.keys((1, 1, S, D), seed=seed))
    V = kvt_synth.bf16_bits(kvt_synth.values((1, 1, S, D), seed=seed + 1))
    q = kvt_synth.bf16_bits(kvt_synth.queries((1, g, D), seed=seed + 2))
    sl = np.array([S], np.int32)
    t0 = time.perf_counter()
    for u in range(n_units):
        s = specs[(u * 7) % L]
        oracle.layer_decode(s.mode, s.key_bits, s.value_bits, s.group, s.residual, K, V, q, sl, 1 / math.sqrt(D))
    dt = time.perf_counter() - t0
    return dt, n_units / (L * H)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2502_04420_b200 as kvt   # only for the config loader (host C, no GPU work)

    specs, desc = layer_specs(args.workload, kvt)
    _, shape, B, S = WORKLOADS[args.workload]
    S = args.ctx or S
    for _ in range(args.warmup):
        oracle_sample(specs, shape, S, 1)
    tot_t, tot_tok = 0.0, 0.0
    for _ in range(args.steps):
        dt, tok = oracle_sample(specs, shape, S, 1)
        tot_t += dt
        tot_tok += tok
    value = tot_tok / tot_t
    sample = (f"per step: 1 (layer, kv head) unit of 1 sequence at S={S} (layers rotate), i.e. 1/{shape[0] * shape[1]} "
              f"of a decode token; oracle = O2 static build + fp64 read-back + fp64 Eq.1 attention")
    line = {"impl": "reference", "metric": "decode tokens/s (attention-only, mixed-precision KV)", "value": value,
            "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (kvt_synth: N(0,1) K with x11 channel outliers, "
            "N(0,1) V, 0.5 N(0,1) q)",
            "config": {"workload": args.workload, "layers": desc, "batch": 1, "ctx": S, "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
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

    specs, desc = layer_specs(args.workload, kvt)
    _, (L, H, Hq), B, S_ctx = WORKLOADS[args.workload]
    B = args.batch or B
    S_ctx = args.ctx or S_ctx
    seqshard = args.workload.endswith("seqshard")
    S0 = S_ctx - 1                                           # prefilled; the first timed append makes S_ctx
    n_steps_total = args.warmup + 2 * args.steps + (0 if args.no_e2e else args.warmup + args.steps)
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
    len0 = torch.zeros(B, dtype=torch.int32, device=dev)
    nS0 = torch.full((B,), S0, dtype=torch.int32, device=dev)
    for l, spec in enumerate(specs):
        if args.paged:        # vLLM-style: one block table per layer, pages assigned in a random order
            pg = torch.Generator().manual_seed(500 + l)
            bt = torch.randperm(B * (cap // 32), generator=pg).view(B, cap // 32).to(torch.int32).to(dev)
            cache = kvt.LayerCache(spec, B, H, D, cap, device=dev, block_table=bt, num_pages=B * (cap // 32))
        else:
            cache = kvt.LayerCache(spec, B, H, D, cap, device=dev)
        gen.manual_seed(1000 * rank + l)
        Kp = torch.randn(B, H, S0, D, device=dev, generator=gen)
        Kp[..., ::8] *= 11.0                                  # kvt_synth recipe: key channel outliers
        Kp = Kp.to(torch.bfloat16)
        Vp = torch.randn(B, H, S0, D, device=dev, generator=gen).to(torch.bfloat16)
        kvt.quantize_append(cache, Kp, Vp, len0, nS0, len_before_host=[0] * B, n_new_host=[S0] * B)
        del Kp, Vp
        torch.cuda.empty_cache()                              # large batches: keep the prefill temporaries from fragmenting HBM
        caches.append(cache)
    torch.cuda.synchronize()
    # ---- per-step inputs (resident): new k, v per layer and q per layer ----
    # one contiguous device buffer of all per-step inputs (q, k_new, v_new of every layer) and one of all
    # outputs, so the end-to-end leg moves them with one host->device and one device->host copy per step
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
    ws_bytes = max(kvt.decode_workspace_bytes(c, Hq, [cap] * B) for c in caches)
    ws = torch.zeros(max(ws_bytes, 16), dtype=torch.uint8, device=dev)      # merge counters start at zero
    n_combine = 0     # the tensor-core kernel merges cut units in-kernel (last CTA); see launches.csv
    len_before = torch.full((B,), S0, dtype=torch.int32, device=dev)
    len_after = torch.full((B,), S0 + (1 if appends else 0), dtype=torch.int32, device=dev)
    ones = torch.ones(B, dtype=torch.int32, device=dev)
    scale = 1.0 / math.sqrt(D)
    stream = torch.cuda.current_stream()
    exch = None
    if seqshard:
        part = torch.empty(B, Hq, D + 2, dtype=torch.float32, device=dev)
        gathered = torch.empty(world, B, Hq, D + 2, dtype=torch.float32, device=dev)
        if args.exchange == "symm":
            from paper_2502_04420_b200.seqshard import SymmExchange

            if world == 1 and not dist.is_initialized():
                dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1,
                                        device_id=dev)
            exch = SymmExchange((B, Hq, D + 2), dev)

    def step(ev=None, bs=0):
        q, k_new, v_new, outs = bufsets[bs]
        for l in range(L):
            if appends:
                kvt.quantize_append(caches[l], k_new[l], v_new[l], len_before, ones, n_new_max=1, stream=stream)
            if ev is not None:
                ev[l][0].record(stream)
            if exch is not None:          # fused exchange: push into the peers' buffers, barrier, combine
                k = exch.k
                kvt.decode_attention_partial_push(caches[l], q[l], len_after, exch.slots[k], scale=scale,
                                                  workspace=ws, stream=stream)
                if ev is not None:
                    ev[l][1].record(stream)
                exch.handle.barrier(channel=0)
                exch.k ^= 1
                kvt.combine_partials(exch.buf[k], out=outs[l], stream=stream)
            elif seqshard:
                kvt.decode_attention_partial(caches[l], q[l], len_after, scale=scale, partial=part, workspace=ws,
                                             stream=stream)
                if ev is not None:
                    ev[l][1].record(stream)
                if world > 1:
                    dist.all_gather_into_tensor(gathered, part)
                else:
                    gathered[0].copy_(part)
                kvt.combine_partials(gathered, out=outs[l], stream=stream)
            else:
                kvt.decode_attention(caches[l], q[l], len_after, scale=scale, out=outs[l], workspace=ws, stream=stream)
                if ev is not None:
                    ev[l][1].record(stream)
        if appends:
            len_before.add_(1)
            len_after.add_(1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # per-layer attention events (live, on the launching stream) for the roofline
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(L)]
           for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    S_first = S0 + (args.warmup + 1 if appends else 0)
    sampler = ClockSampler(dev.index) if not args.profile else None
    if sampler:
        sampler.__enter__()
    # timed region: K steps back to back (no per-layer events: the attention launch may then overlap the
    # tail of the same layer's append, programmatic dependent launch)
    start.record(stream)
    for i in range(args.steps):
        step()
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # roofline pass: the next K steps again, with CUDA events around every attention launch
    for i in range(args.steps):
        step(evs[i])
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    ms = start.elapsed_time(end)
    attn_ms = sum(e[0].elapsed_time(e[1]) for st in evs for e in st)
    if world > 1:
        t = torch.tensor([ms, attn_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, attn_ms = t.tolist()
    ms_per_step = ms / args.steps
    value = world * B / (ms_per_step / 1000.0)

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
                "algorithmic_bytes_per_step": alg / args.steps}

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
                stream.wait_event(h2d_done[j])
                if i >= 2:
                    stream.wait_event(d2h_done[j])           # step i-2's outputs left buffer set j
                step(bs=j)
                comp_done[j].record(stream)
                with torch.cuda.stream(cs):
                    cs.wait_event(comp_done[j])
                    h_out.copy_(d_outs[j], non_blocking=True)    # step i's outputs, device -> host
                    d2h_done[j].record(cs)
            stream.wait_event(d2h_done[(n - 1) % 2])

        e2e_run(args.warmup)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(stream)
        e2e_run(args.steps)
        e2.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ems = s2.elapsed_time(e2)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": world * B / (ems / args.steps / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        n_units = 48
        dt, tok = oracle_sample(specs, (L, H, Hq), S_first, n_units)
        cpu = {"value": tok / dt, "unit": "tokens/s", "cores": 1, "kind": "oracle",
               "sample": f"{n_units} (layer, kv head) units of 1 sequence at S={S_first} (= {tok:.3f} decode tokens, "
                         f"{dt:.1f} s), single-threaded C oracle: O2 static build + fp64 read-back + fp64 Eq.1"}

    clocks = sampler.summary() if sampler else None
    if rank == 0:
        line = {"metric": "decode tokens/s (attention-only, mixed-precision KV)", "value": value, "unit": "tokens/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong" if seqshard else "weak", "vs_baseline": None,
                "dtype": "f32 accumulate of f16 tensor-core products (u2/u4/u8 codes, bf16 in/out)",
                "data": "synthetic (N(0,1) K with x11 outliers on channels c%8==0, N(0,1) V, 0.5 N(0,1) q)",
                "config": {"workload": args.workload, "layers": desc, "shape": {"L": L, "H_kv": H, "H_q": Hq, "d": D},
                           "batch_per_gpu": B, "ctx": f"{S_first}..{S_first + args.steps - 1}",
                           "parallelism": ((f"sequence-sharded x{world} (partial pushed into peer symmetric memory -> barrier -> combine)"
                                            if exch is not None else
                                            f"sequence-sharded x{world} (partial -> NCCL all-gather -> combine)") if seqshard
                                           else f"batch-partitioned x{world} (no collective)"),
                           "l2": "inputs larger than L2 (cache %.1f GB/GPU)" % (sum(c.nbytes for c in caches) / 1e9),
                           "kv_layout": "paged (shuffled 32-token pages, block table)" if args.paged else "dense"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": args.steps * ((1 if appends else 0) * L + L + (L if seqshard else 0) + n_combine),
                "clocks": clocks,
                "gb_per_s_attention": achieved}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_kvt(args)


if __name__ == "__main__":
    main()
