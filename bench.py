#!/usr/bin/env python
"""bench.py -- KVQuant decode hot path on B200: one decode step = for every layer,
quantize-on-append of the new token's (K_preRoPE, V) + decode attention of the query
over the whole compressed cache (the paper's "Total" includes the
packing).

Default workload (N=1): BASELINE config 3, 3-bit: LLaMA-7B shape, 32 layers x 128K
cached tokens, nuq3 with 1% outliers.  Each layer's cache is 447 MB (> 126 MB L2) and
the step walks 32 distinct layers, so every timed iteration streams from HBM (no flush
needed; stated in config.l2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3_nuq3|c3_nuq4|c2|...]
  python bench.py --impl reference ...   # the CPU oracle as the reference arm

N > 1 (torchrun, one process per GPU): the same context is sequence-sharded across the
ranks (pos_base offsets), each rank attends over its shard, partials are all-gathered
over NCCL and merged by the CUDA merge kernel ("scaling": "strong").

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn µs/token & HBM GB/s vs roofline at 128K–10M ctx, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3_nuq3")
    ap.add_argument("--tokens", type=int, default=0, help="override context length")
    ap.add_argument("--layers", type=int, default=0, help="override layer count")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=8192)
    ap.add_argument("--splits", type=int, default=0)
    return ap.parse_args()


def workload(args):
    from kvq_synth import CONFIGS, Workload
    w = CONFIGS[args.workload]
    if args.tokens or args.layers:
        w = Workload(w.name + "-override", args.layers or w.n_layers, w.H_q, w.H_kv, w.d,
                     args.tokens or w.T, w.bits, w.ppm, w.qnorm)
    return w


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ clocks sampler --
class Clocks:
    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace('.', '').isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace('.', '').isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# -------------------------------------------------------------- CPU oracle timing --
def oracle_sample(w, T_s, seed=0):
    """Time the oracle (as it stands) on a bounded sample: one layer, T_s cached tokens:
    one append (quantize 1 token) + one decode attend.  Returns (seconds, threads)."""
    import oracle as O
    from kvq_synth import calib, gen
    D = w.D
    cal = calib.calibrate_layer(gen.gen_keys(seed, 0, 1024, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(seed, 0, 1024, D, stream=gen.STREAM_CAL_V),
                                w.bits, w.ppm, qnorm=w.qnorm)
    K = gen.gen_keys(seed, 0, T_s, D)
    V = gen.gen_values(seed, 0, T_s, D)
    cache = O.prefill(K, V, cal["key_lo"], cal["key_hi"], cal["cbK"], cal["cbV"], w.ppm)
    q = gen.gen_queries(seed, 0, w.H_q, w.H_kv, w.d)[0]
    threads = os.cpu_count() or 1
    kn = gen.gen_keys(seed, 0, 1, D, stream=gen.STREAM_APP_K)[0]
    vn = gen.gen_values(seed, 0, 1, D, stream=gen.STREAM_APP_V)[0]

    def step():
        O.quantize_key(kn, cal["key_lo"], cal["key_hi"], cal["cbK"])
        O.quantize_value(vn, w.ppm, cal["cbV"])
        O.attend_partial(cache, q, T_s, H_q=w.H_q, H_kv=w.H_kv, d=w.d, key_lo=cal["key_lo"],
                         key_hi=cal["key_hi"], cbK_dec=cal["cbK_dec"], cbV_dec=cal["cbV_dec"],
                         nthreads=threads)
    return step, threads


def cpu_baseline(w, T_s, min_seconds=10.0):
    """The oracle as it stands, on a bounded sample: repeat (1 append + 1 attend over T_s
    cached tokens of one layer) until >= min_seconds of CPU work, then scale per token
    and per layer to the workload (linear in both)."""
    step, threads = oracle_sample(w, T_s)
    reps, t0 = 0, time.perf_counter()
    while True:
        step()
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds or reps >= 1000:
            break
    per = dt / reps
    scale = (w.T / T_s) * w.n_layers
    return {"value": per * scale * 1e6, "unit": "us/token", "cores": threads, "kind": "oracle",
            "sample": f"{reps} x (1 append + 1 attend) on 1 layer with {T_s} cached tokens "
                      f"(of {w.T}), fp64 C oracle, OpenMP over heads; per-step time scaled "
                      f"x{w.T}/{T_s} tokens x{w.n_layers} layers (linear in both)",
            "sample_seconds": dt}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    w = workload(args)
    T_s = args.cpu_sample_tokens
    step, threads = oracle_sample(w, T_s)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    scale = (w.T / T_s) * w.n_layers
    v = dt * scale * 1e6
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "us/token",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": v / 1e3, "higher_is_better": False,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "layers": w.n_layers, "context": w.T, "H_q": w.H_q,
                       "H_kv": w.H_kv, "head_dim": w.d, "bits": w.bits, "outlier_ppm": w.ppm},
            "cpu_baseline": {"value": v, "unit": "us/token", "cores": threads, "kind": "oracle",
                             "sample": f"per step: 1 layer, {T_s} cached tokens, 1 append + 1 "
                                       f"attend; scaled x{w.T}/{T_s} x{w.n_layers} layers"},
            "e2e": {"value": v, "unit": "us/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ our arm --
def run_ours(args):
    import torch
    import torch.distributed as dist

    from kvq_synth import calib, gen
    from paper_2401_18079_b200 import accounting, kvq
    from paper_2401_18079_b200.sharding import ShardPlan, gather_partials

    world, rank, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = workload(args)
    plan = ShardPlan(w.T, world, rank)
    e2e_steps = 0 if (args.no_e2e or world > 1) else max(3, args.steps // 2)
    steps_total = args.warmup + args.steps + e2e_steps + 2
    L, D, H, d = w.n_layers, w.D, w.H_q, w.d

    # offline calibration (input preparation; one set of constants for every layer handle)
    cal = calib.calibrate_layer(gen.gen_keys(0, 0, 2048, D, stream=gen.STREAM_CAL_K),
                                gen.gen_values(0, 0, 2048, D, stream=gen.STREAM_CAL_V),
                                w.bits, w.ppm, qnorm=w.qnorm)
    caches = []
    prefill_ms = 0.0
    t_setup = time.time()
    for l in range(L):
        c = kvq.KVQCache(n_q_heads=H, n_kv_heads=w.H_kv, head_dim=d, bits=w.bits,
                         outlier_ppm=w.ppm, capacity_tokens=plan.capacity(steps_total),
                         key_cb=cal["cbK"], val_cb=cal["cbV"], key_cb_dec=cal["cbK_dec"],
                         val_cb_dec=cal["cbV_dec"], key_lo=cal["key_lo"], key_hi=cal["key_hi"],
                         pos_base=plan.pos_base, device=local)
        if args.splits:
            c.set_splits(args.splits)
        n = plan.end - plan.start
        chunk = 1 << 16
        for a in range(0, n, chunk):
            b = min(n, a + chunk)
            Kl = gen.gen_layer_torch(1000 * l + 31 * rank + a, l, b - a, D, dev, "K")
            Vl = gen.gen_layer_torch(1000 * l + 31 * rank + a + 7, l, b - a, D, dev, "V")
            if l == 0:   # a9: time layer 0's prefill quantization (kvq_prefill_quantize)
                pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                pe0.record()
                c.prefill(Kl, Vl)
                pe1.record()
                pe1.synchronize()
                prefill_ms += pe0.elapsed_time(pe1)
            else:
                c.prefill(Kl, Vl)
            del Kl, Vl
        caches.append(c)
    for c in caches:
        c.sync()
    t_setup = time.time() - t_setup

    # per-step inputs: new token (K, V) per layer, pre-RoPE q per layer
    knew = torch.stack([gen.gen_layer_torch(7 + l, l, steps_total, D, dev, "K") for l in range(L)])
    vnew = torch.stack([gen.gen_layer_torch(9 + l, l, steps_total, D, dev, "V") for l in range(L)])
    qsc = torch.tensor(np.repeat(gen.query_scale(0, 0, D, d), H // w.H_kv), dtype=torch.float32,
                       device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    qs = (torch.randn((steps_total, L, H, d), generator=g, device=dev)
          * qsc[None, None, :, None]).half()
    o = torch.zeros((L, H, d), dtype=torch.float32, device=dev)
    part = torch.zeros((L, H, d + 2), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    is_tail = rank == plan.tail_owner
    st = {"pos": w.T, "s": 0}

    def step(kb, vb, qb, ob):
        pos, s = st["pos"], st["s"]
        for l in range(L):
            if is_tail:
                caches[l].append(kb[l, s], vb[l, s], stream)
            if world == 1:
                caches[l].attend(qb[s, l], pos, ob[l], stream)
            else:
                caches[l].attend_partial(qb[s, l], pos, part[l], stream)
                parts = gather_partials(part[l])
                kvq.merge_partials(parts, ob[l], device=local, stream=stream)
        st["pos"], st["s"] = pos + 1, s + 1

    for _ in range(args.warmup):
        step(knew, vnew, qs, o)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with clocks:
        t0.record(stream)
        for _ in range(args.steps):
            step(knew, vnew, qs, o)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    ms_per_step = elapsed_ms / args.steps

    # attend-only pass: per-launch CUDA events on the launching stream
    pos = st["pos"]
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(L * args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(L * args.steps)]
    for s in range(args.steps):
        for l in range(L):
            i = s * L + l
            starts[i].record(stream)
            if world == 1:
                caches[l].attend(qs[s, l], pos, o[l], stream)
            else:
                caches[l].attend_partial(qs[s, l], pos, part[l], stream)
            ends[i].record(stream)
    torch.cuda.synchronize()
    att_ms_mean = float(np.mean([a.elapsed_time(b) for a, b in zip(starts, ends)]))

    # e2e: same step through the public API with pinned HOST buffers; the library
    # stages K, V, q host->device and o device->host inside each call.
    e2e = None
    if e2e_steps:
        kh, vh, qh = knew.cpu().pin_memory(), vnew.cpu().pin_memory(), qs.cpu().pin_memory()
        oh = torch.zeros((L, H, d), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            step(kh, vh, qh, oh)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e = {"value": e2e_ms * 1e3, "unit": "us/token",
               "h2d_bytes_per_step": L * (2 * D * 2 + H * d * 2),
               "d2h_bytes_per_step": L * H * d * 4, "steps": e2e_steps}

    kv = caches[0].info()["value_outliers"]
    Tc = caches[0].num_tokens
    spans = [c.key_outlier_span(0, c.num_tokens) for c in caches]
    nnz_mean = float(np.mean([e - b for b, e in spans]))
    bytes_att = accounting.attend_bytes(Tc, D, w.bits, kv, int(nnz_mean), H, d)
    peak, peak_kind = measured_peaks()
    achieved = bytes_att / (att_ms_mean * 1e-3) / 1e9
    info = caches[0].info()

    # a9 prefill: HBM bytes per token-layer = K, V in (fp16) + codes, (s, z), CSC pointer and
    # outlier records (canonical + bucketed) out; the prefill launches of layer 0, CUDA events
    n_pf = plan.end - plan.start
    pf_bytes = n_pf * (4 * D + 2 * D * w.bits / 8 + 8 + 4 + 8 * (kv + nnz_mean / max(Tc, 1)))
    prefill_line = {"ns_per_token_layer": prefill_ms * 1e6 / max(n_pf, 1), "tokens": n_pf,
                    "gbs": pf_bytes / (prefill_ms * 1e-3) / 1e9 if prefill_ms > 0 else None,
                    "frac": (pf_bytes / (prefill_ms * 1e-3) / 1e9) / peak if prefill_ms > 0 else None,
                    "kernels": "qz_kernel (count) + scan_counts_kernel + qz_kernel (write) + sort_buckets_kernel x2"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(w, args.cpu_sample_tokens)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "unit": "us/token", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_per_step * 1e3, "unit": "us/token",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f16xf16->f32 (u%d codes; quantization decisions f64)" % w.bits,
            "data": "synthetic",
            "config": {"workload": w.name, "layers": L, "context": w.T, "H_q": H, "H_kv": w.H_kv,
                       "head_dim": d, "bits": w.bits, "outlier_ppm": w.ppm,
                       "parallelism": f"seq-shard x{world}" if world > 1 else "single-gpu",
                       "step": "per layer: kvq_append(new K,V) + kvq_decode_attend(q)",
                       "l2": f"inputs larger than L2 ({bytes_att / 1e6:.0f} MB per layer, "
                             f"{L} layers cycled per step)"},
            "attend_us_per_layer": att_ms_mean * 1e3,
            "attend_us_per_step": att_ms_mean * 1e3 * L,
            "hbm_gbs_step": bytes_att * L / (ms_per_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(w.name),
                         "kernel": {1: "att_wa_kernel", 2: "att_wag_kernel"}.get(info.get("attend_kernel"), "att_kernel")
                                   + " (kvq_decode_attend: one launch)",
                         "bytes_per_launch": bytes_att, "peak_kind": peak_kind,
                         "splits": info["splits"], "heads_per_cta": info["heads_per_cta"]},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps * L * (2 if world == 1 else 3),
            "clocks": clocks.summary(),
            "key_outliers_per_token": nnz_mean / max(Tc, 1),
            # effective: step time minus the attend-only time (the attend launched right after
            # an append overlaps its prologue with the append through programmatic dependent
            # launch, so this is below the append kernel's own duration)
            "append_us_per_layer": (ms_per_step - att_ms_mean * L) * 1e3 / L,
            "prefill": prefill_line,
            "setup_s": t_setup,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ncu_traffic(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per attend launch from the committed
    ncu --set full capture (profiles/att_traffic.json), or None if none was taken for this
    workload."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "att_traffic.json")
    try:
        with open(path) as f:
            rec = json.load(f).get(workload)
        return None if rec is None else rec["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
