"""Benchmark: structures/sec for log_partition + marginals (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2a|c1|...] [--all-configs]

Headline workload (BASELINE.json configs[1]): MonotoneAlignmentCRF, batch 256,
src n=512, tgt m=128 (move_potentials [256,513,129,3] fp32 = 203 MB, larger
than L2), log_partition + marginals.  One step = one batched fused
forward-backward launch over the whole batch on device-resident synthetic
N(0,1) inputs (structural -inf as the reference builders place them).

Multi-GPU (torchrun, one rank per GPU): weak scaling -- every rank owns its
own batch of B independent structures (no data-path collective); after each
step the per-structure log Z shard is all-gathered over NCCL so
every rank holds Z for the global batch.  Timing = CUDA events per step,
max over ranks.

`e2e` measures the same metric through the public batched entry
(kernels.nw_fb on host-resident pinned inputs): H2D of the potentials,
the fused kernel, D2H of log Z and marginals, all inside the timed region.

`--impl reference` times the reference algorithm on the host CPU: the
float64 NumPy restatement in oracle/ (the reference itself is Python and
cannot run on the GPU box), over a bounded sample of the same workload with
one worker process per host core.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

NEG_INF = float("-inf")
METRIC = "structures/sec for log_partition+marginals"
FALLBACK_HBM = 6650.0

# per-structure algorithmic work and config shapes.
# bound: "hbm" -> bytes / HBM GB/s; "fp32" -> FLOP / FP32 FMA peak; "mufu" -> MUFU ops / MUFU peak.
CONFIGS = {
    "c1": dict(workload="LinearChainCRF", B=32, shape=dict(n=128, m=32), work=1_040_644, bound="hbm",
               argmax=True, kernel="chain_lin_kernel"),
    "c2a": dict(workload="MonotoneAlignmentCRF", B=256, shape=dict(n=512, m=128), work=1_588_252, bound="hbm",
                argmax=False, kernel="nw_mitm_kernel"),
    "c2b": dict(workload="CTCDist", B=256, shape=dict(T=512, V=128, L=128), work=921_088, bound="mufu",
                argmax=False, kernel="ctc_dir_kernel + ctc_marg_kernel<9>"),
    "c3": dict(workload="SpanningTreeCRF non-projective (Matrix-Tree, multi-root)", B=512, shape=dict(n=128),
               work=4_194_304, bound="fp32", argmax=False, kernel="mtt_kernel<true>"),
    "c4": dict(workload="SpanningTreeCRF projective (Eisner, multi-root) + Kuhlmann argmax", B=256,
               shape=dict(n=128), work=2_504_320, bound="mufu", argmax=True, kernel="eisner_lin_kernel"),
    "c5a": dict(workload="TreeCRF (CKY)", B=128, shape=dict(n=64, m=32), work=790_532, bound="hbm",
                argmax=False, kernel="tree_kernel<1>"),
    "c5b": dict(workload="PCFG (CKY, NT=32, PT=32)", B=128, shape=dict(n=64, NT=32, PT=32),
                work=2_130_444_288, bound="fp32", argmax=False, kernel="pcfg_kernel<1>"),
}
HEADLINE = "c2a"
# e2e: instance slices per request in kernels.run_host_batch (PCIe-bound configs
# overlap H2D, kernels and D2H; tiny batches run as one slice)
E2E_CHUNKS = {"c1": 1, "c2a": [32] * 7 + [24, 8], "c2b": [32] * 7 + [24, 8], "c3": 8, "c4": 4, "c5a": 4, "c5b": 1}
if os.environ.get("SDB_E2E_CHUNKS"):
    E2E_CHUNKS = {k: json.loads(os.environ["SDB_E2E_CHUNKS"]) for k in E2E_CHUNKS}
# nominal B200 compute peaks (not in MEASURED_PEAKS.json): 148 SM x 128 FMA lanes x 2 x 1.965 GHz;
# MUFU ex2 148 x 16 x 1.965 GHz
NOMINAL = {"fp32": (74_440.0, "GFLOP/s"), "mufu": (4_653.0, "Gop/s")}


def _rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", FALLBACK_HBM)), "measured"
    return FALLBACK_HBM, "fallback"


def _traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(cfg_name)
    return None


# ------------------------------------------------------------------ inputs


def _spanning_dev(torch, B, n, device, g):
    adj = torch.randn(B, n + 1, n + 1, device=device, generator=g)
    adj[:, :, 0] = NEG_INF
    i = torch.arange(n + 1, device=device)
    adj[:, i, i] = NEG_INF
    return adj


def make_inputs(cfg, device, seed):
    """Synthetic N(0,1) inputs with the reference builders' structural -inf
    (tests/golden/builders.py mirrors helpers.py:12-87)."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    c = CONFIGS[cfg]
    B, sh = c["B"], c["shape"]
    if cfg == "c1":
        return (torch.randn(B, sh["m"], device=device, generator=g),
                torch.randn(B, sh["n"] - 1, sh["m"], sh["m"], device=device, generator=g))
    if cfg == "c2a":
        th = torch.randn(B, sh["n"] + 1, sh["m"] + 1, 3, device=device, generator=g)
        th[:, 0, :, 0] = NEG_INF
        th[:, 0, :, 1] = NEG_INF
        th[:, :, 0, 0] = NEG_INF
        th[:, :, 0, 2] = NEG_INF
        return (th,)
    if cfg == "c2b":
        return (torch.randn(B, sh["T"], sh["V"], device=device, generator=g),
                torch.randint(1, sh["V"], (B, sh["L"]), device=device, generator=g, dtype=torch.int32))
    if cfg in ("c3", "c4"):
        return (_spanning_dev(torch, B, sh["n"], device, g),)
    if cfg == "c5a":
        return (torch.randn(B, sh["n"], sh["n"], sh["m"], device=device, generator=g),)
    if cfg == "c5b":
        nt, pt, n = sh["NT"], sh["PT"], sh["n"]
        root = torch.log_softmax(torch.randn(B, nt, device=device, generator=g), -1)
        rules = torch.log_softmax(torch.randn(B, nt, (nt + pt) ** 2, device=device, generator=g), -1)
        rules = rules.view(B, nt, nt + pt, nt + pt)
        emis = torch.randn(B, n, pt, device=device, generator=g)
        return (root, rules, emis)
    raise KeyError(cfg)


def step_fn(cfg, inputs):
    """One step = log_partition + marginals (+ argmax where the config lists
    it) over the whole batch; returns the outputs (logz first)."""
    from paper_2308_03291_b200 import kernels as K

    if cfg == "c1":
        def f():
            (lz, mi, mt, st), (tags, _, _) = K.chain_fb_viterbi(inputs[0], inputs[1], True)
            return lz, mi, mt, tags
        return f
    if cfg == "c2a":
        return lambda: K.nw_fb(inputs[0], True)[:2]
    if cfg == "c2b":
        return lambda: K.ctc_fb(inputs[0], inputs[1], True)[:2]
    if cfg == "c3":
        return lambda: K.mtt(inputs[0], False, True)[:2]
    if cfg == "c4":
        def f():
            (lz, mg, st), (heads, _, _) = K.eisner_kuhlmann(inputs[0], False, True)
            return lz, mg, heads
        return f
    if cfg == "c5a":
        return lambda: K.tree_fb(inputs[0], True)[:2]
    if cfg == "c5b":
        return lambda: K.pcfg_fb(inputs[0], inputs[1], inputs[2], None, True)[:2]
    raise KeyError(cfg)


def kernel_fn(cfg, inputs):
    """The dominant launch alone (for the roofline)."""
    from paper_2308_03291_b200 import kernels as K

    return {
        "c1": lambda: K.chain_fb(inputs[0], inputs[1], True),
        "c2a": lambda: K.nw_fb(inputs[0], True),
        "c2b": lambda: K.ctc_fb(inputs[0], inputs[1], True),
        "c3": lambda: K.mtt(inputs[0], False, True),
        "c4": lambda: K.eisner(inputs[0], False, True),
        "c5a": lambda: K.tree_fb(inputs[0], True),
        "c5b": lambda: K.pcfg_fb(inputs[0], inputs[1], inputs[2], None, True),
    }[cfg]


def launches_per_step(cfg):
    return {"c1": 4, "c2a": 1, "c2b": 2, "c3": 1, "c4": 3, "c5a": 4, "c5b": 1}[cfg]


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML every
    millisecond (the headline region is only ~12 ms long), nvidia-smi every
    200 ms if NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event / throttle-reason bits
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, [reason names])
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _sample(self):
        if self._nvml is not None:
            nv, h = self._nvml
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((float(sm), float(mx), [k for k, v in self.BITS.items() if bits & v]))
                return
            except Exception:
                self._nvml = None
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            vals = [v.strip() for v in out.stdout.strip().split(",")]
            if len(vals) == 6 and vals[0].replace(".", "").isdigit():
                names = list(self.BITS)
                self.samples.append((float(vals[0]), float(vals[1]),
                                     [names[k] for k in range(4) if vals[2 + k].lower() == "active"]))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.001 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------------ ours


def measure_config(cfg, device, rank, world, steps, warmup, clocks=False):
    """Time `steps` batched steps (CUDA events per step, L2 flushed between
    steps when the inputs fit in L2), the dominant kernel alone, and the
    end-to-end host->device->host path.  Returns a dict of ms figures."""
    import torch
    import torch.distributed as dist

    c = CONFIGS[cfg]
    B = c["B"]
    inputs = make_inputs(cfg, device, seed=1000 + rank)
    fn = step_fn(cfg, inputs)
    kfn = kernel_fn(cfg, inputs)
    from paper_2308_03291_b200.sharding import gather_shards

    def step():
        out = fn()
        if world > 1:  # the only collective: log Z shards -> every rank
            gather_shards(out[0], world * B)
        return out

    in_bytes = sum(t.numel() * t.element_size() for t in inputs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device) if in_bytes < (160 << 20) else None
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    # Single GPU: replay the step (and the dominant launch) as CUDA graphs, so a
    # step's host-side launch cost (ctypes, output allocation, several launches on
    # two streams) never shows up as GPU idle time inside an event pair.
    if world == 1:
        step, kfn = _graphed(step, torch, device), _graphed(kfn, torch, device)
    stream = torch.cuda.current_stream(device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(device.index) if clocks else None
    if clk:
        clk.__enter__()
    for e0, e1 in evs:
        if flush is not None:
            flush.zero_()
        e0.record(stream)
        step()
        e1.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if world > 1:
        dist.barrier()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps
    # dominant kernel alone: launches queued back to back (no host sync in
    # between, so host-side launch overhead never shows up as GPU idle time
    # inside an event pair)
    kev = []
    for _ in range(max(3, min(steps, 10))):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        kfn()
        e1.record(stream)
        kev.append((e0, e1))
    torch.cuda.synchronize()
    kt = [e0.elapsed_time(e1) for e0, e1 in kev]
    kms = sum(kt) / len(kt)
    # e2e: pinned host inputs -> H2D -> fused kernels -> D2H of log Z and marginals
    host_in = [t.cpu().pin_memory() for t in inputs]
    probe = [o for o in fn() if o is not None]
    host_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in probe]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(o.numel() * o.element_size() for o in host_out)
    from paper_2308_03291_b200 import kernels as K

    et = []
    # the host path (pinned copies, launches, syncs) needs a longer warm-up than the device
    # loop: per-step e2e times keep falling for the first ~15 iterations
    ew = max(warmup, 20)
    for it in range(ew + steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        # public host-batch entry: H2D / kernels / D2H of instance slices overlapped
        K.run_host_batch(lambda *d: step_fn(cfg, d)(), host_in, host_out, device, chunks=E2E_CHUNKS.get(cfg, 1))
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= ew:
            et.append(e0.elapsed_time(e1))
    if os.environ.get("SDB_E2E_DEBUG"):
        print("[bench] e2e ms per step", [round(x, 2) for x in et], file=sys.stderr)
    e2e_ms = sum(et) / len(et)
    t = torch.tensor([ms, kms, e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kms, e2e_ms = t.tolist()
    return dict(ms=ms, kms=kms, e2e_ms=e2e_ms, h2d=h2d, d2h=d2h, clocks=clk.summary() if clk else None,
                l2="flushed between steps" if flush is not None else "inputs larger than L2")


def _graphed(fn, torch, device):
    """fn captured once into a CUDA graph (same kernels, same device buffers);
    falls back to the eager callable if capture is not possible."""
    try:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device)
        s.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(s):
            fn()  # warm the allocator on the capture stream
        torch.cuda.current_stream(device).wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g.replay
    except Exception as e:  # pragma: no cover - capture is an optimisation
        print("[bench] graph capture failed (%s); timing eager launches" % e, file=sys.stderr)
        return fn


def roofline(cfg, kms):
    c = CONFIGS[cfg]
    B = c["B"]
    if c["bound"] == "hbm":
        peak, src = _peaks()
        ach = B * c["work"] / (kms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": _traffic(cfg), "kernel": c["kernel"], "kernel_ms": round(kms, 4), "peak_source": src,
                "algorithmic_bytes_per_structure": c["work"]}
    peak, unit = NOMINAL[c["bound"]]
    ach = B * c["work"] / (kms / 1e3) / 1e9
    return {"bound": c["bound"], "achieved": round(ach, 1), "peak": peak, "unit": unit, "frac": round(ach / peak, 4),
            "traffic": _traffic(cfg), "kernel": c["kernel"], "kernel_ms": round(kms, 4),
            "peak_source": "nominal (148 SM x 1.965 GHz)", "algorithmic_work_per_structure": c["work"]}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _rank_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    cfg = args.config
    c = CONFIGS[cfg]
    B = c["B"]
    r = measure_config(cfg, device, rank, world, args.steps, args.warmup, clocks=True)
    value = world * B / (r["ms"] / 1e3)
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "structures/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32 potentials; fp32/fp64 log accumulators",
        "data": "synthetic N(0,1) log-potentials (seeded), structural -inf per reference builders",
        "config": {"workload": c["workload"], "batch_per_gpu": B, "global_batch": world * B, **c["shape"],
                   "parallelism": f"batch-dp{world}", "l2": r["l2"],
                   "step": "log_partition + marginals" + (" + argmax" if c["argmax"] else "")},
        "e2e": {"value": round(world * B / (r["e2e_ms"] / 1e3), 2), "unit": "structures/s",
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]},
        "gpu_launches": launches_per_step(cfg) * args.steps,
        "roofline": roofline(cfg, r["kms"]),
        "clocks": r["clocks"],
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    if args.all_configs:
        others = {}
        for oc in CONFIGS:
            if oc == cfg:
                continue
            print(f"[bench] measuring {oc}", file=sys.stderr, flush=True)
            ro = measure_config(oc, device, rank, world, max(3, args.steps // 2), 3)
            oo = CONFIGS[oc]
            entry = {"workload": oo["workload"], "batch_per_gpu": oo["B"], **oo["shape"],
                     "value": round(world * oo["B"] / (ro["ms"] / 1e3), 2), "unit": "structures/s",
                     "ms_per_step": round(ro["ms"], 4),
                     "e2e_value": round(world * oo["B"] / (ro["e2e_ms"] / 1e3), 2),
                     "roofline": roofline(oc, ro["kms"])}
            if rank == 0 and world == 1 and not args.no_cpu:
                print(f"[bench] cpu baseline {oc}", file=sys.stderr, flush=True)
                cb = cpu_baseline(oc, budget_s=args.cpu_budget / 3)
                entry["cpu_baseline"] = cb
                if cb["value"]:
                    entry["speedup_vs_cpu"] = round(entry["value"] / cb["value"], 1)
            others[oc] = entry
        line["configs"] = others
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------- CPU baseline


def _worker_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"


def _cpu_worker(task):
    """One instance of the workload through the float64 oracle restatement
    (log_partition + marginals [+ argmax]); returns its compute seconds."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cfg, seed = task
    import numpy as np
    from golden import builders as bld
    from oracle import sd_oracle as O

    sh = CONFIGS[cfg]["shape"]
    if cfg == "c1":
        init, tr = bld.chain(seed, sh["n"], sh["m"])
        t0 = time.perf_counter()
        O.chain_marginals(init[None], tr[None])
        O.chain_viterbi(init[None], tr[None])
    elif cfg == "c2a":
        th = bld.alignment(seed, sh["n"], sh["m"])
        t0 = time.perf_counter()
        O.nw_marginals(th)
    elif cfg == "c2b":
        fp, tg = bld.ctc(seed, sh["T"], sh["V"], sh["L"])
        t0 = time.perf_counter()
        O.ctc_marginals(fp[None], np.array([tg]))
    elif cfg == "c3":
        adj = bld.spanning(seed, sh["n"])
        t0 = time.perf_counter()
        O.mtt_log_partition(adj)
        O.mtt_marginals(adj)
    elif cfg == "c4":
        adj = bld.spanning(seed, sh["n"])
        t0 = time.perf_counter()
        O.eisner_marginals(adj)
        O.kuhlmann_heads(adj)
    elif cfg == "c5a":
        th = bld.tree(seed, sh["n"], sh["m"])
        t0 = time.perf_counter()
        O.tree_marginals(th)
    elif cfg == "c5b":
        r, ru, e = bld.pcfg(seed, sh["n"], sh["NT"], sh["PT"])
        t0 = time.perf_counter()
        O.pcfg_span_marginals(r, ru, e)  # log-space, splits batched (reference: 163 s per instance)
    else:
        raise KeyError(cfg)
    return time.perf_counter() - t0


def cpu_baseline(cfg, budget_s=15.0):
    """The oracle port timed on all host cores: a bounded sample of
    instances of the same workload, one worker process per core."""
    cores = os.cpu_count() or 1
    if CONFIGS[cfg].get("cpu_skip"):
        return {"value": None, "unit": "structures/s", "cores": cores, "kind": "port",
                "sample": "skipped: " + CONFIGS[cfg]["cpu_skip"]}
    one = _cpu_worker((cfg, 0))  # warm + size the sample
    per_core = max(1, int(budget_s / max(one, 1e-6) / 2))
    k = min(cores * per_core, CONFIGS[cfg]["B"] * 4)
    if one > budget_s:  # a single instance exceeds the budget (PCFG): time one instance per core
        k = cores
    # spawn (not fork): the parent holds a CUDA context and helper threads
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_worker_init) as pool:
        pool.map(_cpu_worker, [(cfg, 0)] * cores, chunksize=1)  # warm every worker (imports, BLAS init)
        t0 = time.perf_counter()
        pool.map_async(_cpu_worker, [(cfg, 1000 + i) for i in range(k)], chunksize=1).get(timeout=20 * budget_s + 60)
        wall = time.perf_counter() - t0
    return {"value": round(k / wall, 4), "unit": "structures/s", "cores": cores, "kind": "port",
            "sample": f"{k} instances of {CONFIGS[cfg]['workload']} (seeds 1000..{1000 + k - 1}), "
                      f"oracle/sd_oracle.py float64 NumPy, {cores} worker processes, wall {wall:.2f}s"}


def run_reference(args):
    rank, world, _ = _rank_env()
    if rank != 0:
        return
    cfg = args.config
    vals = []
    for _ in range(min(args.warmup, 1)):
        cpu_baseline(cfg, budget_s=args.cpu_budget / 4)
    base = None
    for _ in range(args.steps):
        base = cpu_baseline(cfg, budget_s=args.cpu_budget)
        vals.append(base["value"])
    v = sum(vals) / len(vals)
    c = CONFIGS[cfg]
    line = {
        "metric": METRIC, "value": round(v, 3), "unit": "structures/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(c["B"] / v * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1) (seeded)",
        "config": {"workload": c["workload"], "batch_per_gpu": c["B"], **c["shape"]},
        "impl": "reference",
        "cpu_baseline": {**base, "value": round(v, 3)},
        "e2e": {"value": round(v, 3), "unit": "structures/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--all-configs", action="store_true", help="also measure every other BASELINE config")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
