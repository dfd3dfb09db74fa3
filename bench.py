"""Benchmark: structures/sec for log_partition + marginals (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2a|c1|...] [--scaling weak|strong] [--all-configs]

Headline workload (BASELINE.json configs[1]): MonotoneAlignmentCRF, batch 256,
src n=512, tgt m=128 (move_potentials [256,513,129,3] fp32 = 203 MB, larger
than L2), log_partition + marginals.  One step = one batched fused
forward-backward launch over the whole batch on device-resident synthetic
N(0,1) inputs (structural -inf as the reference builders place them).

Multi-GPU: one process per GPU (torchrun, or `--gpus N` spawns the N ranks
itself); every rank runs its shard through the sharding entry
(paper_2308_03291_b200/sharding.py) and the per-structure log Z / status are
all-gathered over NCCL.  `--scaling weak` (default): every rank
owns the config's batch; `--scaling strong`: the config's batch is split over
the ranks.  Timing = CUDA events per step, max over ranks.

`e2e` is the same metric through the batched entry on HOST-resident pinned
inputs (H2D of the potentials, the fused kernels, D2H of log Z and
marginals, all inside the timed region); `e2e_api` goes through the
reference-shaped Python API (`sd.batch_map(sd.log_partition, dists)` +
`sd.batch_map(sd.marginals, dists)` on float64 NumPy distribution objects).

`--impl reference` times the UNMODIFIED reference (`structdist` 0.1.0 from
/root/reference/pkg installed into baseline/_ref) through its public calls
`sd.log_partition(d); sd.marginals(d)` (+ `sd.argmax(d)` where the config
lists it) on the host cores, one worker process per core, a bounded sample
of the same workload per step.  If baseline/_ref is absent it falls back to
the float64 NumPy restatement in oracle/ and says so (`kind: port`).
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
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

NEG_INF = float("-inf")
METRIC = "structures/sec for log_partition+marginals"
FALLBACK_HBM = 6650.0
L2_BYTES = 126 << 20

# per-structure algorithmic work and config shapes.
# bound: "hbm" -> bytes / HBM GB/s; "fp32"/"fp64" -> FLOP / FMA peak; "mufu" -> MUFU ops / MUFU peak.
CONFIGS = {
    "c1": dict(workload="LinearChainCRF", B=32, shape=dict(n=128, m=32), work=1_040_644, bound="hbm",
               argmax=True, kernel="chain_lin_kernel", in_bytes=32 * (32 + 127 * 32 * 32) * 4),
    "c2a": dict(workload="MonotoneAlignmentCRF", B=256, shape=dict(n=512, m=128), work=1_588_252, bound="hbm",
                argmax=False, kernel="nw_mitm_kernel", in_bytes=256 * 513 * 129 * 3 * 4),
    "c2b": dict(workload="CTCDist", B=256, shape=dict(T=512, V=128, L=128), work=921_088, bound="mufu",
                argmax=False, kernel="ctc_dir_kernel + ctc_marg_kernel<9>", in_bytes=256 * 512 * 128 * 4),
    "c3": dict(workload="SpanningTreeCRF non-projective (Matrix-Tree, multi-root)", B=512, shape=dict(n=128),
               work=4_194_304, bound="fp64", argmax=False, kernel="mtt_kernel<double,true,false>",
               in_bytes=512 * 129 * 129 * 4),
    "c4": dict(workload="SpanningTreeCRF projective (Eisner, multi-root) + Kuhlmann argmax", B=256,
               shape=dict(n=128), work=2_504_320, bound="mufu", argmax=True, kernel="eisner_lin_kernel",
               in_bytes=256 * 129 * 129 * 4),
    "c5a": dict(workload="TreeCRF (CKY)", B=128, shape=dict(n=64, m=32), work=790_532, bound="hbm",
                argmax=False, kernel="tree_fold + tree_lin + tree_emit", in_bytes=128 * 64 * 64 * 32 * 4),
    "c5b": dict(workload="PCFG (CKY, NT=32, PT=32)", B=128, shape=dict(n=64, NT=32, PT=32),
                work=2_130_444_288, bound="fp32", argmax=False, kernel="pcfg_kernel<1>",
                in_bytes=128 * (32 + 32 * 64 * 64 + 64 * 32) * 4),
}
HEADLINE = "c2a"
# e2e: instance slices per request in kernels.run_host_batch (PCIe-bound configs
# overlap H2D, kernels and D2H; tiny batches run as one slice)
E2E_CHUNKS = {"c1": 1, "c2a": [32] * 7 + [24, 8], "c2b": 8, "c3": 4, "c4": 2, "c5a": 4, "c5b": 1}  # tools/e2e_sweep_cfg.py
# the unmodified reference takes ~170 s per C5b instance: its arm uses the port there
REF_TOO_SLOW = {"c5b": "reference PCFG marginals take ~170 s per instance (SURVEY.md §6)"}


def _rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    """Roofline denominators: HBM from the driver's MEASURED_PEAKS.json; FP32 /
    FP64 FMA and MUFU ex2 from tools/micro/peaks.cu run on a B200
    (profiles/peaks_r02.json)."""
    out = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            out["hbm"] = (float(json.load(f).get("hbm_gbs", FALLBACK_HBM)), "GB/s", "measured (MEASURED_PEAKS.json)")
    else:
        out["hbm"] = (FALLBACK_HBM, "GB/s", "fallback (B200_PROFILING.md)")
    with open(os.path.join(ROOT, "profiles", "peaks_r02.json")) as f:
        pk = json.load(f)
    src = "measured (tools/micro/peaks.cu, profiles/peaks_r02.json)"
    out["fp32"] = (pk["fp32_ffma_gflops"], "GFLOP/s", src)
    out["fp64"] = (pk["fp64_dfma_gflops"], "GFLOP/s", src)
    out["mufu"] = (pk["mufu_ex2_gops"], "Gop/s", src)
    return out


def _traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(cfg_name)
    return None


def config_dict(cfg, world, scaling):
    """The workload description -- identical in both arms."""
    c = CONFIGS[cfg]
    B = c["B"]
    per_gpu = B if scaling == "weak" else -(-B // world)
    glob = B * world if scaling == "weak" else B
    return {"workload": c["workload"], "batch_per_gpu": per_gpu, "global_batch": glob, **c["shape"],
            "parallelism": f"batch-dp{world}", "scaling": scaling,
            "l2": "inputs larger than L2" if c["in_bytes"] > L2_BYTES else "flushed between steps",
            "step": "log_partition + marginals" + (" + argmax" if c["argmax"] else "")}


# ------------------------------------------------------------------ inputs


def _spanning_dev(torch, B, n, device, g):
    adj = torch.randn(B, n + 1, n + 1, device=device, generator=g)
    adj[:, :, 0] = NEG_INF
    i = torch.arange(n + 1, device=device)
    adj[:, i, i] = NEG_INF
    return adj


def make_inputs(cfg, device, seed, B=None):
    """Synthetic N(0,1) inputs with the reference builders' structural -inf
    (tests/golden/builders.py mirrors helpers.py:12-87)."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    c = CONFIGS[cfg]
    B, sh = (c["B"] if B is None else B), c["shape"]
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
    it) over the batch; returns the outputs (logz first, status last)."""
    from paper_2308_03291_b200 import kernels as K

    if cfg == "c1":
        def f():
            (lz, mi, mt, st), (tags, _, _) = K.chain_fb_viterbi(inputs[0], inputs[1], True)
            return lz, mi, mt, tags, st
        return f
    if cfg == "c2a":
        return lambda: K.nw_fb(inputs[0], True)
    if cfg == "c2b":
        return lambda: K.ctc_fb(inputs[0], inputs[1], True)
    if cfg == "c3":
        return lambda: K.mtt(inputs[0], False, True)
    if cfg == "c4":
        def f():
            (lz, mg, st), (heads, _, _) = K.eisner_kuhlmann(inputs[0], False, True)
            return lz, mg, heads, st
        return f
    if cfg == "c5a":
        return lambda: K.tree_fb(inputs[0], True)
    if cfg == "c5b":
        return lambda: K.pcfg_fb(inputs[0], inputs[1], inputs[2], None, True)
    raise KeyError(cfg)


def kernel_fn(cfg, inputs):
    """The dominant launch(es) alone (for the roofline)."""
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
    millisecond (the headline region is only ~10 ms long), nvidia-smi every
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


def _host_dists(cfg, B, seed0):
    """The same workload as reference-shaped float64 host distribution objects
    (builders.py, seeds seed0 + i) for the Python-API e2e."""
    import paper_2308_03291_b200 as sd
    from golden import builders as bld

    sh = CONFIGS[cfg]["shape"]
    out = []
    for i in range(B):
        s = seed0 + i
        if cfg == "c1":
            out.append(sd.LinearChainCRF(*bld.chain(s, sh["n"], sh["m"])))
        elif cfg == "c2a":
            out.append(sd.MonotoneAlignmentCRF(bld.alignment(s, sh["n"], sh["m"])))
        elif cfg == "c2b":
            fp, tg = bld.ctc(s, sh["T"], sh["V"], sh["L"])
            out.append(sd.CTCDist(fp, tg))
        elif cfg == "c3":
            out.append(sd.SpanningTreeCRF(bld.spanning(s, sh["n"])))
        elif cfg == "c4":
            out.append(sd.SpanningTreeCRF(bld.spanning(s, sh["n"]), projective=True))
        elif cfg == "c5a":
            out.append(sd.TreeCRF(bld.tree(s, sh["n"], sh["m"])))
        elif cfg == "c5b":
            out.append(sd.PCFG(*bld.pcfg(s, sh["n"], sh["NT"], sh["PT"])))
    return out


def measure_config(cfg, device, rank, world, steps, warmup, scaling="weak", clocks=False, api=True):
    """Time `steps` batched steps (CUDA events per step, L2 flushed between
    steps when the inputs fit in L2), the dominant kernel alone, and the
    end-to-end host->device->host paths.  Returns a dict of ms figures
    (max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2308_03291_b200 import kernels as K
    from paper_2308_03291_b200.sharding import gather_shards, shard_range

    c = CONFIGS[cfg]
    Bg = c["B"] * world if scaling == "weak" else c["B"]
    a, b = shard_range(Bg, world, rank)
    inputs = make_inputs(cfg, device, seed=1000 + rank, B=b - a)
    fn = step_fn(cfg, inputs)
    kfn = kernel_fn(cfg, inputs)

    def step():
        out = fn()
        if world > 1:  # the only collective: log Z / status shards -> every rank
            gather_shards(out[0], Bg)
            gather_shards(out[-1], Bg)
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
    # dominant kernel alone: launches queued back to back
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
    # e2e: pinned host inputs -> sharding entry (H2D of this rank's slice) -> fused kernels ->
    # D2H of log Z and marginals, every step
    host_in = [t.cpu().pin_memory() for t in inputs]
    probe = [o for o in fn() if o is not None]
    host_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in probe]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(o.numel() * o.element_size() for o in host_out)
    et = []
    ew = max(warmup, 20)  # the host path needs a longer warm-up than the device loop
    for it in range(ew + steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        # H2D / kernels / D2H of instance slices overlapped (kernels.run_host_batch)
        K.run_host_batch(lambda *d: step_fn(cfg, d)(), host_in, host_out, device, chunks=E2E_CHUNKS.get(cfg, 1))
        if world > 1:
            gather_shards(torch.as_tensor(host_out[0]).to(device), Bg)
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= ew:
            et.append(e0.elapsed_time(e1))
    e2e_ms = sum(et) / len(et)
    # the reference-shaped Python API on float64 host distribution objects (this rank's shard)
    api_ms = None
    if api:
        dists = _host_dists(cfg, b - a, 5000 + a)
        import paper_2308_03291_b200 as sd

        at = []
        for it in range(2 + max(2, min(steps, 5))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sd.batch_map(sd.log_partition, dists)
            sd.batch_map(sd.marginals, dists)
            if c["argmax"]:
                sd.batch_map(sd.argmax, dists)
            torch.cuda.synchronize()
            if it >= 2:
                at.append((time.perf_counter() - t0) * 1e3)
        api_ms = sum(at) / len(at)
    t = torch.tensor([ms, kms, e2e_ms, api_ms or 0.0], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kms, e2e_ms, api_ms = t.tolist()
    return dict(ms=ms, kms=kms, e2e_ms=e2e_ms, api_ms=api_ms if api else None, h2d=h2d, d2h=d2h, Bg=Bg,
                local=b - a, clocks=clk.summary() if clk else None)


def roofline(cfg, kms, local_B):
    c = CONFIGS[cfg]
    peak, unit, src = _peaks()[c["bound"]]
    ach = local_B * c["work"] / (kms / 1e3) / 1e9
    key = "algorithmic_bytes_per_structure" if c["bound"] == "hbm" else "algorithmic_work_per_structure"
    return {"bound": c["bound"], "achieved": round(ach, 1), "peak": peak, "unit": unit, "frac": round(ach / peak, 4),
            "traffic": _traffic(cfg), "kernel": c["kernel"], "kernel_ms": round(kms, 4), "peak_source": src,
            key: c["work"], "structures_per_launch": local_B}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _rank_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    cfg = args.config
    c = CONFIGS[cfg]
    r = measure_config(cfg, device, rank, world, args.steps, args.warmup, args.scaling, clocks=True,
                       api=not args.no_api)
    Bg = r["Bg"]
    line = {
        "metric": METRIC,
        "value": round(Bg / (r["ms"] / 1e3), 2),
        "unit": "structures/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 4),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "fp32 potentials; fp32/fp64 accumulators" + ("; fp64 elimination" if cfg == "c3" else ""),
        "data": "synthetic N(0,1) log-potentials (seeded), structural -inf per reference builders",
        "config": config_dict(cfg, world, args.scaling),
        "e2e": {"value": round(Bg / (r["e2e_ms"] / 1e3), 2), "unit": "structures/s",
                "h2d_bytes_per_step": r["h2d"] * world, "d2h_bytes_per_step": r["d2h"] * world,
                "path": "kernels.run_host_batch on pinned host slices (H2D, kernels, D2H overlapped)"},
        "gpu_launches": launches_per_step(cfg) * args.steps,
        "roofline": roofline(cfg, r["kms"], r["local"]),
        "clocks": r["clocks"],
    }
    if r["api_ms"]:
        line["e2e_api"] = {"value": round(Bg / (r["api_ms"] / 1e3), 2), "unit": "structures/s",
                           "path": "sd.batch_map(sd.log_partition) + sd.batch_map(sd.marginals)"
                                   + (" + sd.batch_map(sd.argmax)" if c["argmax"] else "")
                                   + " on float64 NumPy distribution objects (host conversion included)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
        if not args.no_ref_sample:
            line["cpu_reference"] = reference_sample(cfg)
    if args.all_configs:
        others = {}
        for oc in CONFIGS:
            if oc == cfg:
                continue
            print(f"[bench] measuring {oc}", file=sys.stderr, flush=True)
            ro = measure_config(oc, device, rank, world, max(3, args.steps // 2), 3, args.scaling,
                                api=not args.no_api)
            entry = {**config_dict(oc, world, args.scaling),
                     "value": round(ro["Bg"] / (ro["ms"] / 1e3), 2), "unit": "structures/s",
                     "ms_per_step": round(ro["ms"], 4),
                     "e2e_value": round(ro["Bg"] / (ro["e2e_ms"] / 1e3), 2),
                     "roofline": roofline(oc, ro["kms"], ro["local"])}
            if ro["api_ms"]:
                entry["e2e_api_value"] = round(ro["Bg"] / (ro["api_ms"] / 1e3), 2)
            if rank == 0 and world == 1 and not args.no_cpu:
                print(f"[bench] cpu baseline {oc}", file=sys.stderr, flush=True)
                cb = cpu_baseline(oc, budget_s=args.cpu_budget / 3)
                entry["cpu_baseline"] = cb
                if cb["value"]:
                    entry["speedup_vs_cpu"] = round(entry["value"] / cb["value"], 1)
                if not args.no_ref_sample and oc not in REF_TOO_SLOW:
                    entry["cpu_reference"] = reference_sample(oc)
            others[oc] = entry
        line["configs"] = others
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------- CPU baselines


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


def _ref_dist(sd, cfg, seed):
    from golden import builders as bld

    sh = CONFIGS[cfg]["shape"]
    if cfg == "c1":
        return sd.LinearChainCRF(*bld.chain(seed, sh["n"], sh["m"]))
    if cfg == "c2a":
        return sd.MonotoneAlignmentCRF(bld.alignment(seed, sh["n"], sh["m"]))
    if cfg == "c2b":
        fp, tg = bld.ctc(seed, sh["T"], sh["V"], sh["L"])
        return sd.CTCDist(fp, tg)
    if cfg == "c3":
        return sd.SpanningTreeCRF(bld.spanning(seed, sh["n"]))
    if cfg == "c4":
        return sd.SpanningTreeCRF(bld.spanning(seed, sh["n"]), projective=True)
    if cfg == "c5a":
        return sd.TreeCRF(bld.tree(seed, sh["n"], sh["m"]))
    if cfg == "c5b":
        return sd.PCFG(*bld.pcfg(seed, sh["n"], sh["NT"], sh["PT"]))
    raise KeyError(cfg)


def _ref_worker(task):
    """One instance through the UNMODIFIED reference's public calls
    (dist.py:68-163): sd.log_partition + sd.marginals (+ sd.argmax)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cfg, seed = task
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import structdist as sd

    d = _ref_dist(sd, cfg, seed)
    t0 = time.perf_counter()
    sd.log_partition(d)
    sd.marginals(d)
    if CONFIGS[cfg]["argmax"]:
        sd.argmax(d)
    return time.perf_counter() - t0


def _have_reference():
    return os.path.isdir(os.path.join(REF_PATH, "structdist"))


def _pool_rate(worker, cfg, k, cores, seed0, timeout):
    """structures/s of k instances (seeds seed0..) on `cores` worker processes
    (warmed first); returns (rate, wall seconds)."""
    ctx = mp.get_context("spawn")  # the parent may hold a CUDA context
    with ctx.Pool(cores, initializer=_worker_init) as pool:
        pool.map(_cpu_probe, [worker.__name__] * cores, chunksize=1)  # imports + BLAS init in every worker
        t0 = time.perf_counter()
        pool.map_async(worker, [(cfg, seed0 + i) for i in range(k)], chunksize=1).get(timeout=timeout)
        wall = time.perf_counter() - t0
    return k / wall, wall


def _cpu_probe(name):
    """Warm a worker: import the code path it will time."""
    if name == "_ref_worker":
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        import structdist  # noqa: F401
    else:
        from oracle import sd_oracle  # noqa: F401
    return 0


def cpu_baseline(cfg, budget_s=15.0):
    """The oracle port (float64 NumPy restatement, oracle/sd_oracle.py) timed
    on all host cores: a bounded sample of the same workload."""
    cores = os.cpu_count() or 1
    one = _cpu_worker((cfg, 0))  # warm + size the sample
    per_core = max(1, int(budget_s / max(one, 1e-6) / 2))
    k = min(cores * per_core, CONFIGS[cfg]["B"] * 4)
    if one > budget_s:  # a single instance exceeds the budget (PCFG): time one instance per core
        k = cores
    rate, wall = _pool_rate(_cpu_worker, cfg, k, cores, 1000, 20 * budget_s + 60)
    return {"value": round(rate, 4), "unit": "structures/s", "cores": cores, "kind": "port",
            "sample": f"{k} instances of {CONFIGS[cfg]['workload']} (seeds 1000..{1000 + k - 1}), "
                      f"oracle/sd_oracle.py float64 NumPy, {cores} worker processes, wall {wall:.2f}s"}


def reference_sample(cfg):
    """The unmodified reference (baseline/_ref) on one round of instances
    (one per host core) -- the kind of number the reference arm reports."""
    cores = os.cpu_count() or 1
    if not _have_reference():
        return {"value": None, "kind": "reference", "sample": "baseline/_ref not installed"}
    if cfg in REF_TOO_SLOW:
        return {"value": None, "kind": "reference", "sample": "skipped: " + REF_TOO_SLOW[cfg]}
    k = cores if CONFIGS[cfg]["B"] >= cores else CONFIGS[cfg]["B"]
    rate, wall = _pool_rate(_ref_worker, cfg, k, cores, 1000, 3600)
    return {"value": round(rate, 4), "unit": "structures/s", "cores": cores, "kind": "reference",
            "sample": f"{k} instances (seeds 1000..{1000 + k - 1}) through structdist 0.1.0 (baseline/_ref) "
                      f"sd.log_partition + sd.marginals" + (" + sd.argmax" if CONFIGS[cfg]["argmax"] else "")
                      + f", {cores} worker processes, wall {wall:.2f}s"}


def run_reference(args):
    """The reference arm: rank 0 times the unmodified reference on the host
    cores (each step: one bounded sample of the workload); other ranks exit."""
    rank, world, _ = _rank_env()
    if rank != 0:
        return
    cfg = args.config
    c = CONFIGS[cfg]
    cores = os.cpu_count() or 1
    use_ref = _have_reference() and cfg not in REF_TOO_SLOW
    worker = _ref_worker if use_ref else _cpu_worker
    if use_ref:
        # one instance per core per step for the slow families; whole batches for the fast ones
        one_est = {"c1": 0.03, "c3": 0.03, "c5a": 0.3, "c4": 2.5, "c2a": 10.0, "c2b": 18.0}.get(cfg, 10.0)
        k = max(cores, min(c["B"], int(cores * max(1.0, 2.0 / one_est))))
    else:
        k = cores
    vals, walls = [], []
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_worker_init) as pool:
        pool.map(_cpu_probe, [worker.__name__] * cores, chunksize=1)
        for it in range(min(args.warmup, 1) + args.steps):
            t0 = time.perf_counter()
            pool.map_async(worker, [(cfg, 1000 + (it * k + i) % max(c["B"], k)) for i in range(k)],
                           chunksize=1).get(timeout=3600)
            wall = time.perf_counter() - t0
            if it >= min(args.warmup, 1):
                vals.append(k / wall)
                walls.append(wall)
    v = len(vals) / sum(1.0 / x for x in vals)  # structures / total wall
    kind = "reference" if use_ref else "port"
    what = ("structdist 0.1.0 (unmodified, baseline/_ref) sd.log_partition + sd.marginals"
            + (" + sd.argmax" if c["argmax"] else "") if use_ref
            else "oracle/sd_oracle.py float64 NumPy restatement" + (
                f" (reference skipped: {REF_TOO_SLOW[cfg]})" if cfg in REF_TOO_SLOW else " (baseline/_ref absent)"))
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "structures/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(c["B"] / v * 1e3, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1) (seeded)",
        "config": config_dict(cfg, world, args.scaling),
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 4), "unit": "structures/s", "cores": cores, "kind": kind,
                         "sample": f"{k} instances per step x {args.steps} steps, {what}, {cores} worker "
                                   f"processes, step walls {min(walls):.2f}-{max(walls):.2f}s"},
        "e2e": {"value": round(v, 4), "unit": "structures/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main


def _spawned(rank, world, port, argv):
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    main(argv)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--all-configs", action="store_true", help="also measure every other BASELINE config")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ref-sample", action="store_true", help="skip the unmodified-reference sample in our arm")
    ap.add_argument("--no-api", action="store_true", help="skip the Python-API e2e")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher: spawn one rank per GPU ourselves (same env contract as torchrun)
        import torch.multiprocessing as tmp

        port = 29400 + os.getpid() % 2000
        tmp.start_processes(_spawned, args=(args.gpus, port, argv if argv is not None else sys.argv[1:]),
                            nprocs=args.gpus, start_method="spawn")
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
