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

# per-structure algorithmic bytes and the config shapes
CONFIGS = {
    "c1": dict(workload="LinearChainCRF", B=32, n=128, m=32, bytes=1_040_644, bound="hbm",
               kernel="chain_fwd_bwd_kernel", note="chain forward-backward (+ marginal pass)"),
    "c2a": dict(workload="MonotoneAlignmentCRF", B=256, n=512, m=128, bytes=1_588_252, bound="hbm",
                kernel="nw_kernel<1>", note="fused backward + forward-with-marginals"),
}


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


def make_inputs(cfg, device, seed):
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    c = CONFIGS[cfg]
    if cfg == "c2a":
        th = torch.randn(c["B"], c["n"] + 1, c["m"] + 1, 3, device=device, generator=g)
        th[:, 0, :, 0] = NEG_INF
        th[:, 0, :, 1] = NEG_INF
        th[:, :, 0, 0] = NEG_INF
        th[:, :, 0, 2] = NEG_INF
        return (th,)
    if cfg == "c1":
        return (torch.randn(c["B"], c["m"], device=device, generator=g),
                torch.randn(c["B"], c["n"] - 1, c["m"], c["m"], device=device, generator=g))
    raise KeyError(cfg)


def step_fn(cfg, inputs):
    from paper_2308_03291_b200 import kernels as K

    if cfg == "c2a":
        return lambda: K.nw_fb(inputs[0], True)
    if cfg == "c1":
        return lambda: K.chain_fb(inputs[0], inputs[1], True)
    raise KeyError(cfg)


def launches_per_step(cfg):
    return {"c2a": 1, "c1": 2}[cfg]


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ ours


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
    inputs = make_inputs(cfg, device, seed=1000 + rank)
    fn = step_fn(cfg, inputs)
    gathered = torch.empty(world * B, dtype=torch.float64, device=device)

    def step():
        out = fn()
        if world > 1:
            dist.all_gather_into_tensor(gathered, out[0])
        return out

    # L2 flush buffer (inputs of small configs fit in the 126 MB L2)
    in_bytes = sum(t.numel() * t.element_size() for t in inputs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device) if in_bytes < (160 << 20) else None

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e0, e1 in evs:
            if flush is not None:
                flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = [e0.elapsed_time(e1) for e0, e1 in evs]  # ms per step
    ms = sum(times) / len(times)
    # kernel-only duration of the dominant launch (no collective) for the roofline
    kt = []
    for _ in range(max(3, args.steps)):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        kt.append(e0.elapsed_time(e1))
    kms = sum(kt) / len(kt)

    # e2e through the public batched entry with host pinned buffers
    host_in = [t.cpu().pin_memory() for t in inputs]
    probe = [o for o in fn() if o is not None and o.dtype != torch.int32]
    host_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in probe]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(o.numel() * o.element_size() for o in host_out)
    e2e_times = []
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        dev_in = [t.to(device, non_blocking=True) for t in host_in]
        out = [o for o in step_fn(cfg, dev_in)() if o is not None and o.dtype != torch.int32]
        for h, o in zip(host_out, out):
            h.copy_(o, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = sum(e2e_times) / len(e2e_times)

    t = torch.tensor([ms, kms, e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kms, e2e_ms = t.tolist()
    value = world * B / (ms / 1e3)
    peak, peak_kind = _peaks()
    achieved = B * c["bytes"] / (kms / 1e3) / 1e9
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "structures/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32 (fp64 log accumulators)",
        "data": "synthetic N(0,1) log-potentials (seeded), structural -inf per reference builders",
        "config": {"workload": c["workload"], "batch_per_gpu": B, "global_batch": world * B,
                   **{k: c[k] for k in ("n", "m")}, "parallelism": f"batch-dp{world}",
                   "l2": "flushed between steps" if flush is not None else "inputs larger than L2"},
        "e2e": {"value": round(world * B / (e2e_ms / 1e3), 2), "unit": "structures/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step(cfg) * args.steps,
        "roofline": {"bound": c["bound"], "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": _traffic(cfg),
                     "kernel": c["kernel"], "kernel_ms": round(kms, 4), "peak_source": peak_kind,
                     "algorithmic_bytes_per_structure": c["bytes"]},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------- CPU baseline


def _cpu_worker(task):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cfg, seed = task
    from golden import builders as bld
    from oracle import sd_oracle as O

    c = CONFIGS[cfg]
    if cfg == "c2a":
        th = bld.alignment(seed, c["n"], c["m"])
        t0 = time.perf_counter()
        O.nw_marginals(th)
        return time.perf_counter() - t0
    if cfg == "c1":
        init, tr = bld.chain(seed, c["n"], c["m"])
        t0 = time.perf_counter()
        O.chain_marginals(init[None], tr[None])
        return time.perf_counter() - t0
    raise KeyError(cfg)


def cpu_baseline(cfg, budget_s=15.0):
    """Oracle port timed on all host cores: a bounded sample of instances of
    the same workload, one worker process per core."""
    cores = os.cpu_count() or 1
    one = _cpu_worker((cfg, 0))  # warm + size the sample
    per_core = max(1, int(budget_s / max(one, 1e-6) / 2))
    k = min(cores * per_core, CONFIGS[cfg]["B"] * 4)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=os.environ.setdefault, initargs=("OPENBLAS_NUM_THREADS", "1")) as pool:
        t0 = time.perf_counter()
        pool.map(_cpu_worker, [(cfg, 1000 + i) for i in range(k)], chunksize=1)
        wall = time.perf_counter() - t0
    return {"value": round(k / wall, 3), "unit": "structures/s", "cores": cores, "kind": "port",
            "sample": f"{k} instances of {CONFIGS[cfg]['workload']} (seeds 1000..{1000 + k - 1}), "
                      f"oracle/sd_oracle.py float64 NumPy, {cores} worker processes, wall {wall:.2f}s"}


def run_reference(args):
    rank, world, _ = _rank_env()
    if rank != 0:
        return
    cfg = args.config
    vals = []
    for _ in range(args.warmup):
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
        "config": {"workload": c["workload"], "batch_per_gpu": c["B"], "n": c["n"], "m": c["m"]},
        "impl": "reference",
        "cpu_baseline": {**base, "value": round(v, 3)},
        "e2e": {"value": round(v, 3), "unit": "structures/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2a", choices=sorted(CONFIGS))
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
