#!/usr/bin/env python
"""LONGER encoder training-step throughput on B200 (BASELINE.json metric).

metric: samples/sec of fwd+bwd at L=2000 (config 2: B=256/GPU, d=32, K=4 → D=128, k=32
recent queries + m=3 globals, 1 cross + N=2 self layers, InnerTrans merge), whole job.

A step = forward + backward (+ NCCL gradient allreduce when N>1) + Adam, through the C ABI
(`longer_forward_backward`, `longer_adam_step`), captured in one CUDA graph.  `value` times the
device step with CUDA events (inputs resident in HBM, L2 flushed between steps); `e2e` times the
same step with the batch copied from pinned host memory and the loss read back every step.
The per-kernel times behind `roofline` / `kernels` / `sections` come from CUDA events recorded
around the fused kernels in a second capture of the same step, replayed (L2 flushed) after each
timed step and outside its events: the event-record nodes are full dependencies and would
otherwise add their own cost to `ms_per_step`.

`--impl reference` times the CPU reference algorithm (the float64 oracle port of longrec in
oracle/, one single-threaded worker process per host core) on a bounded sample of the same step.

Launch: python bench.py [--gpus N --steps K --warmup W]; with N > 1 and no torchrun environment the
script relaunches itself under torch.distributed.run (one rank per GPU, NCCL); the step is then
routed through paper_2505_04421_b200.dp.DataParallel (two gradient buckets, the first reduced on a
communication stream beside the front-end backward).  `--config c4` measures serving instead.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2_inner": dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner"),
    "c2_concat": dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="concat"),
    "c1": dict(L=256, d=16, K=4, k=16, N=1, m=3),
    "c5_inner": dict(L=10000, d=32, K=8, k=32, N=4, m=3, merge_mode="inner"),
    "c4": dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner"),   # serving on c2 weights
}


def flops_per_sample(cfg) -> int:
    """6 × the reference's exact forward MAC count (pkg/src/longrec/analysis.py:152-171):
    2 FLOP/MAC × (forward + 2 × backward)."""
    d, D, F = cfg.d, cfg.D, cfg.feat_width
    q, v = cfg.k + cfg.m, cfg.merged_len + cfg.m
    n_events = cfg.L
    total = n_events * (F * d + 4 * d * D)
    total += F * d + 2 * d * D + cfg.m * 4 * D * D
    if cfg.merge_mode == "inner":
        Lp = cfg.L_padded
        total += cfg.inner_layers * (12 * Lp * d * d + 2 * Lp * cfg.K * d)
    total += 10 * q * D * D + 2 * v * D * D + 2 * q * v * D
    total += cfg.N * (12 * q * D * D + 2 * q * q * D)
    total += (4 * D + 2 * d) * cfg.head_hidden + cfg.head_hidden
    return 6 * total


def serve_macs(cfg):
    """(cache build MACs per user, scoring MACs per candidate): the reference's exact model,
    muladds_cache_build / muladds_incremental (pkg/src/longrec/analysis.py:174-198)."""
    d, D, F = cfg.d, cfg.D, cfg.feat_width
    q, v = cfg.k + cfg.m - 1, cfg.merged_len + cfg.m - 1
    hh = (4 * D + 2 * d) * cfg.head_hidden + cfg.head_hidden
    build = cfg.L * (F * d + 4 * d * D) + d * D + (cfg.m - 1) * 4 * D * D
    if cfg.merge_mode == "inner":
        build += cfg.inner_layers * (12 * cfg.L_padded * d * d + 2 * cfg.L_padded * cfg.K * d)
    build += 10 * q * D * D + 2 * v * D * D + 2 * q * v * D + cfg.N * (12 * q * D * D + 2 * q * q * D)
    v1, vs = cfg.merged_len + cfg.m, cfg.k + cfg.m
    inc = F * d + d * D + 4 * D * D + 12 * D * D + 2 * v1 * D + cfg.N * (12 * D * D + 2 * vs * D) + hh
    return build, inc


def run_serving(args):
    """--config c4 (BASELINE config 4): c2 weights, per-user KV cache built once, then `--cands`
    candidates per user scored against it; `--users` users per call.  value = cached candidates/s
    (cache and candidate ids resident in HBM, L2 flushed between steps); e2e = the same through
    serving.score_candidates from a pinned host id array with the probabilities read back."""
    import numpy as np
    import torch
    from paper_2505_04421_b200 import ModelConfig, serving as S, synthetic_batch
    from paper_2505_04421_b200.model import LongerModel
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = ModelConfig(**CONFIGS["c2_inner"]).validate()
    U, C = args.users, args.cands
    model = LongerModel(cfg, seed=0)
    users = synthetic_batch(cfg, U, seed=3).to("cuda")
    times = [0] * U
    cand_host = torch.from_numpy(np.random.default_rng(5).integers(0, cfg.vocab, (U, C)).astype(np.int32)).pin_memory()
    cand_dev = cand_host.to("cuda")
    cache = S.build_caches_batch(model, users, times)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(steps):
            flush.fill_(i & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / steps

    probs = torch.empty((U, C), dtype=torch.float32, device="cuda")
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    ms_build = timed(lambda: S.build_caches_batch(model, users, times), args.steps, args.warmup)
    ms_score = timed(lambda: S.score_device(model, cache, cand_dev, probs), args.steps, args.warmup)
    host_out = torch.empty((U, C), dtype=torch.float32).pin_memory()

    def e2e_step():
        p = S.score_candidates(model, cache, cand_host, check=False)      # pinned host ids
        host_out.copy_(p, non_blocking=True)
    ms_e2e = timed(e2e_step, args.steps, args.warmup)
    clk = clocks.stop()
    # parity beside the number: cached scores vs this library's full forward of the same pairs
    n = min(C, 256)
    full = S.full_batch_for(users, cand_dev[0, :n], user=0)
    p_full = model.forward(full)
    dmax = float((probs[0, :n] - p_full).abs().max())
    burst, sustained, hbm, src = peaks()
    b_macs, inc_macs = serve_macs(cfg)
    value = U * C / (ms_score / 1e3)
    achieved = value * 2 * inc_macs / 1e12
    line = {
        "metric": "cached candidates/sec at L=2000 (c4 serving)", "value": value, "unit": "candidates/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_score,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "c4", **CONFIGS["c2_inner"], "users_per_call": U, "candidates_per_user": C,
                   "l2": "flushed between steps"},
        "cache_build": {"users_per_s": U / (ms_build / 1e3), "ms_per_call": ms_build,
                        "tflops": U * 2 * b_macs / (ms_build / 1e3) / 1e12,
                        "cache_bytes_per_user": S.cache_size_bytes(model, 1)},
        "roofline": {"bound": "tensor", "kernel": "cache_score (whole call)", "achieved": achieved, "peak": burst,
                     "unit": "TFLOP/s", "frac": achieved / burst, "traffic": None, "peak_source": src,
                     "flop_per_candidate": 2 * inc_macs},
        "e2e": {"value": U * C / (ms_e2e / 1e3), "unit": "candidates/s", "h2d_bytes_per_step": U * C * 4,
                "d2h_bytes_per_step": U * C * 4, "ms_per_step": ms_e2e},
        "parity": {"max_abs_cached_minus_full_forward": dmax, "pairs": n},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_serving_entry(cfg, C)
    print(json.dumps(line), flush=True)


def cpu_serving_entry(cfg, C):
    """The reference's serving algorithm on the host: oracle/serving_oracle.py (float64
    build_cache + score_with_cache, pinned to the reference's own cached scores) for one user
    and C candidates, all BLAS threads."""
    from oracle import serving_oracle as SO
    from oracle.cpu_pool import cpu_model_name
    from paper_2505_04421_b200 import init_params, synthetic_batch
    import numpy as np
    P = init_params(cfg, 0)
    user = synthetic_batch(cfg, 1, seed=3).as_dict()
    cand = np.random.default_rng(5).integers(0, cfg.vocab, (1, C))
    t0 = time.perf_counter()
    cache = SO.build_cache(P, cfg, user)
    t1 = time.perf_counter()
    SO.score(P, cfg, cache, cand)
    t2 = time.perf_counter()
    return {"value": C / (t2 - t1), "unit": "candidates/s", "cores": os.cpu_count(), "kind": "port",
            "cpu_model": cpu_model_name(), "cache_build_s_per_user": t1 - t0,
            "sample": f"1 user: float64 build_cache ({t1 - t0:.2f} s) + score_with_cache of {C} candidates "
                      f"({t2 - t1:.2f} s), oracle/serving_oracle.py, one process, all BLAS threads"}


def phase_flops(cfg, B):
    """Algorithmic FLOPs of one launch of each probed fused kernel (recompute and padding excluded),
    from the same MAC model as flops_per_sample."""
    d, D, F, L = cfg.d, cfg.D, cfg.feat_width, cfg.L
    q, v = cfg.k + cfg.m, cfg.merged_len + cfg.m
    mlp = L * (F * d + 4 * d * D)
    inner = cfg.inner_layers * (12 * cfg.L_padded * d * d + 2 * cfg.L_padded * cfg.K * d) \
        if cfg.merge_mode == "inner" else 0
    attn = 2 * q * v * D
    return {"fe_fwd": 2 * B * (mlp + inner), "fe_inner_bwd": 4 * B * inner, "fe_mlp_bwd": 4 * B * mlp,
            "xattn_fwd": 2 * B * attn, "xattn_bwd": 4 * B * attn}


def count_graph_kernels(graph):
    """Kernel nodes of the captured step graph, split into ours (longer::) and others."""
    try:
        from cuda.bindings import driver as drv
        g = drv.CUgraph(graph.raw_cuda_graph())
        err, _, n = drv.cuGraphGetNodes(g, 0)
        err, nodes, n = drv.cuGraphGetNodes(g, n)
        ours = other = 0
        for node in nodes[:n]:
            err, t = drv.cuGraphNodeGetType(node)
            if t != drv.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
                continue
            err, prm = drv.cuGraphKernelNodeGetParams(node)
            err, name = drv.cuFuncGetName(prm.func)
            nm = name.decode() if isinstance(name, bytes) else str(name)
            if "longer" in nm:
                ours += 1
            else:
                other += 1
        return ours, other
    except Exception as exc:  # pragma: no cover
        return None, repr(exc)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled (every 20 ms) during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = None

    def start(self):
        import tempfile
        self.out = tempfile.TemporaryFile(mode="w+")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)                      # first sample before the timed region starts

    def stop(self):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = []
        if self.out is not None:
            self.out.seek(0)
            rows = [[x.strip() for x in line.split(",")] for line in self.out.read().splitlines() if line.strip()]
        good = [r for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        sm = sorted(float(r[0]) for r in good)
        mx = [float(r[1]) for r in good if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in good for i, n in enumerate(names) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(good)}


def cpu_samples_default() -> int:
    return 4 * (os.cpu_count() or 1)


def cpu_pool_rate(cfg, n_samples: int, steps: int = 1, warmup: int = 1, seed: int = 1):
    """The reference algorithm on the host's cores: the float64 oracle port of longrec (pinned to
    the reference's own outputs, tests/test_oracle.py), one single-threaded worker process per
    core, each step = fwd + bwd of n_samples sharded over the workers + gradient sum + Adam
    (oracle/cpu_pool.py).  Returns (samples/s over the timed steps, seconds per step, workers)."""
    from oracle.cpu_pool import CpuPool
    from paper_2505_04421_b200 import synthetic_batch
    pool = CpuPool(cfg)
    try:
        for i in range(warmup):
            pool.step(synthetic_batch(cfg, n_samples, seed=seed + i).as_dict())
        total = 0.0
        for i in range(steps):
            batch = synthetic_batch(cfg, n_samples, seed=seed + warmup + i).as_dict()
            t0 = time.perf_counter()
            pool.step(batch)
            total += time.perf_counter() - t0
    finally:
        pool.close()
    return n_samples * steps / total, total / steps, pool.workers


def cpu_baseline_entry(cfg, n_samples, steps, warmup):
    from oracle.cpu_pool import cpu_model_name
    rate, sec, workers = cpu_pool_rate(cfg, n_samples, steps, warmup)
    return {"value": rate, "unit": "samples/s", "cores": workers, "kind": "port",
            "cpu_model": cpu_model_name(), "threads_per_worker": 1,
            "sample": f"{n_samples} samples/step ({sec:.2f} s/step, {steps} timed steps): fwd+bwd of the float64 "
                      f"oracle port of longrec sharded over {workers} single-threaded worker processes, "
                      f"gradient sum, Adam"}


def run_reference(args, cfg):
    """--impl reference: the reference's CPU algorithm (the oracle port) on all host cores, on the
    same config and metric; rank 0 only under torchrun."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if args.config == "c4":
        base = cpu_serving_entry(cfg, args.cands)
        v = base["value"]
        print(json.dumps({"impl": "reference", "metric": "cached candidates/sec at L=2000 (c4 serving)",
                          "value": v, "unit": "candidates/s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
                          "ms_per_step": 1e3 * args.cands / v, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": "c4", **CONFIGS["c4"], "candidates_per_user": args.cands},
                          "cpu_baseline": base,
                          "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    n = args.cpu_samples or cpu_samples_default()
    base = cpu_baseline_entry(cfg, n, args.steps, args.warmup)
    value = base["value"]
    line = {
        "impl": "reference", "metric": "samples/sec fwd+bwd at L=2000", "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, **CONFIGS[args.config], "samples_per_step": n},
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: start N ranks (one per GPU) on this node
    with the same arguments, NCCL init logging on, and return their exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2_inner", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=256, help="samples per GPU per step")
    ap.add_argument("--cpu-samples", type=int, default=0, help="CPU arm samples per step (0: 4 x cores)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--users", type=int, default=64, help="c4: users per serving call")
    ap.add_argument("--cands", type=int, default=512, help="c4: candidates per user")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2505_04421_b200 import ModelConfig
    cfg = ModelConfig(**CONFIGS[args.config]).validate()
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.config == "c4":
        run_serving(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', '1')}")

    import torch
    import torch.distributed as dist
    from paper_2505_04421_b200 import synthetic_batch
    from paper_2505_04421_b200.model import Adam, LongerModel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's init lines (rank / nranks / transport) on the log, for the rank-count check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    B = args.batch
    model = LongerModel(cfg, seed=0, device=str(dev))
    opt = Adam(model, cfg.lr)
    # a few distinct synthetic batches, resident in HBM; host pinned copies for e2e
    n_batches = 4
    host = [synthetic_batch(cfg, B, seed=100 + rank * 17 + i).pin() for i in range(n_batches)]
    dev_batches = [h.to(dev) for h in host]
    static = synthetic_batch(cfg, B, seed=1).to(dev)          # graph input slot
    static2 = synthetic_batch(cfg, B, seed=2).to(dev)         # second slot (e2e double buffering)

    def load(b):
        for f in type(b).FIELDS:
            getattr(static, f).copy_(getattr(b, f), non_blocking=True)

    from paper_2505_04421_b200.dp import DataParallel
    dpm = DataParallel(model) if world > 1 else None

    def step_body(batch=None):
        b = static if batch is None else batch
        if dpm is not None:            # shard's fwd+bwd, early-bucket allreduce beside the front-end bwd
            dpm.loss_backward(b, check=False)
        else:
            model.loss_backward(b, check=False)
        opt.step()

    stream = torch.cuda.current_stream(dev)
    # timing probes around the fused kernels (event records).  An event-record node is a full
    # dependency and costs a few µs, so the timed step graph carries none: the probes live in a
    # second capture of the same step, replayed (L2 flushed) right after each timed step, outside
    # its ms_per_step events.
    import ctypes
    from paper_2505_04421_b200 import _lib as L_
    probe_ev = {}
    for name, ph in L_.PROBES.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); e1.record(stream)            # materialise the events
        probe_ev[name] = (e0, e1)

    def set_probes(on):
        for name, ph in L_.PROBES.items():
            e0, e1 = probe_ev[name]
            L_.check(model._lib.longer_set_probe(ph, ctypes.c_void_p(e0.cuda_event if on else None),
                                                 ctypes.c_void_p(e1.cuda_event if on else None)))
    def mark(msg):
        if os.environ.get("BENCH_TRACE"):
            print(f"[bench] {msg}", file=sys.stderr, flush=True)

    # warm-up (eager) — also sets kernel attributes before capture
    mark("eager warm-up")
    for i in range(2):
        load(dev_batches[i % n_batches])
        step_body()
    torch.cuda.synchronize()
    graph = graph2 = graph_p = None
    graph_note = "disabled (--no-graph)" if args.no_graph else "captured"
    if not args.no_graph:
        mark("capture")
        try:
            s = torch.cuda.Stream(dev)
            s.wait_stream(stream)
            with torch.cuda.stream(s):
                step_body()
            stream.wait_stream(s)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(graph):
                step_body()
            torch.cuda.synchronize()
            # the same step reading the second input slot: the e2e loop alternates slots, so the H2D
            # of step i+1 lands directly in the slot the next graph reads (no device-side copy)
            graph2 = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(graph2):
                step_body(static2)
            torch.cuda.synchronize()
            set_probes(True)
            graph_p = torch.cuda.CUDAGraph(keep_graph=True)      # the same step with the probes
            with torch.cuda.graph(graph_p):
                step_body()
            set_probes(False)
            torch.cuda.synchronize()
            for g in (graph, graph2, graph_p):
                if hasattr(g, "instantiate"):
                    g.instantiate()
        except Exception as exc:          # e.g. a collective that refuses capture: run eagerly
            set_probes(False)
            graph = graph2 = graph_p = None
            graph_note = f"capture failed, eager steps ({type(exc).__name__}: {exc})"[:300]
            print(f"[bench] rank {rank}: {graph_note}", file=sys.stderr, flush=True)
            torch.cuda.synchronize()

    def run_step(slot=0):
        if graph is not None:
            (graph if slot == 0 else graph2).replay()
        else:
            step_body(static if slot == 0 else static2)

    def run_probe_step():
        if graph_p is not None:
            graph_p.replay()
        else:
            set_probes(True)
            step_body()
            set_probes(False)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    for i in range(args.warmup):
        load(dev_batches[i % n_batches])
        run_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    mark("graph warm-up done")
    # ---------------- timed region: device step, inputs resident, L2 flushed between steps
    clocks = ClockSampler(local)
    if not os.environ.get("BENCH_NO_CLOCKS"):
        clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    from cuda.bindings import runtime as rt
    phase_ms = {k: 0.0 for k in probe_ev}
    for i in range(args.steps):
        load(dev_batches[i % n_batches])
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        run_step()
        ev[i][1].record(stream)
        flush.fill_((i + 128) & 0xFF)
        run_probe_step()                            # the kernel probes (outside ev[i])
        torch.cuda.synchronize()
        for k, (e0, e1) in probe_ev.items():
            err, t = rt.cudaEventElapsedTime(e0.cuda_event, e1.cuda_event)
            if int(err) == 0:
                phase_ms[k] += t
            elif i == 0 and rank == 0:
                print(f"probe {k}: {err}", file=sys.stderr)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        dist.barrier()
    mark("timed region done")
    clk = clocks.stop()
    mark("clocks stopped")

    # ---------------- e2e: pinned host batch → H2D, step, loss D2H, every step
    # The usual input pipeline: step i+1's batch is copied host→device on a copy stream while step
    # i runs, into the second of two input slots (one captured graph per slot, so no device-side
    # copy), and the host reads step i's loss (pinned D2H) once step i+1 is queued.
    # One span from before the first H2D to after the last loss read, so every copy is inside it.
    copy_stream = torch.cuda.Stream(dev)
    stage = [static, static2]
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [None, None]
    loss_host = torch.zeros(args.steps, dtype=torch.float32).pin_memory()
    loss_ev = [torch.cuda.Event() for _ in range(args.steps)]
    h2d_bytes = host[0].nbytes()

    def h2d(i):
        slot = stage[i % 2]
        with torch.cuda.stream(copy_stream):
            if consumed[i % 2] is not None:
                copy_stream.wait_event(consumed[i % 2])
            for f in type(slot).FIELDS:
                getattr(slot, f).copy_(getattr(host[i % n_batches], f), non_blocking=True)
            copied[i % 2].record(copy_stream)

    losses = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_start, e2e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_start.record(stream)
    copy_stream.wait_stream(stream)
    h2d(0)
    for i in range(args.steps):
        if i + 1 < args.steps:
            h2d(i + 1)
        stream.wait_event(copied[i % 2])
        mark(f"e2e {i} loaded")
        run_step(i % 2)
        consumed[i % 2] = torch.cuda.Event()                # the step has read its slot
        consumed[i % 2].record(stream)
        mark(f"e2e {i} replayed")
        loss_host[i : i + 1].copy_(model._loss.view(1), non_blocking=True)
        loss_ev[i].record(stream)
        if i > 0:
            loss_ev[i - 1].synchronize()
            losses.append(float(loss_host[i - 1]))
    e2e_end.record(stream)
    e2e_end.synchronize()
    losses.append(float(loss_host[args.steps - 1]))
    mark("e2e synced")
    e2e_ms = e2e_start.elapsed_time(e2e_end)
    if not all(math.isfinite(x) for x in losses):
        raise RuntimeError(f"non-finite loss in the e2e run: {losses}")

    t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(t[0]), float(t[1])
    samples = world * B * args.steps
    value = samples / (ms / 1e3)
    e2e_value = samples / (e2e_ms / 1e3)
    ms_step = ms / args.steps

    if rank == 0:
        burst, sustained, hbm, src = peaks()
        fps = flops_per_sample(cfg)
        achieved = value / world * fps / 1e12
        pf = phase_flops(cfg, B)
        kern_ms = {k: v for k, v in phase_ms.items() if k in pf}         # sections are not kernels
        dom = max(kern_ms, key=lambda k: kern_ms[k]) if kern_ms else None
        kernels, sections = {}, {}
        for k, tms in phase_ms.items():
            if k not in pf:
                if tms > 0:
                    sections[k] = {"ms": tms / args.steps, "share_of_step": tms / args.steps / ms_step}
                continue
            if tms > 0:
                avg = tms / args.steps
                kernels[k] = {"ms_per_launch": avg, "tflops": pf[k] / (avg / 1e3) / 1e12,
                              "share_of_step": avg / ms_step}
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as fh:
                traffic = json.load(fh).get(args.config, {}).get(dom)
        except Exception:
            pass
        n_ours, n_other = count_graph_kernels(graph) if graph is not None else (None, None)
        line = {
            "metric": "samples/sec fwd+bwd at L=2000", "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": args.config, **CONFIGS[args.config], "global_batch": world * B,
                       "per_gpu_batch": B, "parallelism": f"dp{world}", "l2": "flushed between steps",
                       "step": "fwd+bwd+allreduce+adam" if world > 1 else "fwd+bwd+adam",
                       "cuda_graph": graph is not None, "cuda_graph_note": graph_note,
                       "kernel_probes": "kernels / sections timed with CUDA events in a probe-instrumented "
                                        "capture of the same step, replayed (L2 flushed) after each timed step; "
                                        "ms_per_step excludes them"},
            "roofline": ({"bound": "tensor", "kernel": dom, "achieved": kernels[dom]["tflops"], "peak": burst,
                          "unit": "TFLOP/s", "frac": kernels[dom]["tflops"] / burst, "traffic": traffic,
                          "peak_source": src, "ms_per_launch": kernels[dom]["ms_per_launch"],
                          "flop_per_launch": pf[dom]} if dom in kernels else None),
            "roofline_step": {"bound": "tensor", "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
                              "frac": achieved / burst, "peak_source": src,
                              "scope": "whole step, algorithmic FLOPs = 6 x analysis.muladds_full_forward/sample",
                              "frac_of_sustained": achieved / sustained if sustained else None},
            "kernels": kernels,
            "sections": sections,
            "gpu_launches": (n_ours * args.steps) if n_ours is not None else None,
            "gpu_launches_per_step": {"ours": n_ours, "torch_or_nccl": n_other},
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": 4, "ms_per_step": e2e_ms / args.steps,
                    "pipeline": "pinned H2D of step i+1 on a copy stream (into the other of two graph input slots) overlaps step i; loss of every step "
                                "read on the host; one span from the first H2D to the last loss read"},
            "clocks": clk,
        }
        if not args.no_cpu_baseline and world == 1:
            try:
                line["cpu_baseline"] = cpu_baseline_entry(cfg, args.cpu_samples or cpu_samples_default(), 2, 1)
            except Exception as exc:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "error": str(exc)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
