#!/usr/bin/env python
"""Benchmark: sorted keys/s of the B200 LearnedSort (AIPS2o) on BASELINE.json's configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

Default workload (N=1) = the largest single-GPU configuration of
BASELINE.json: C5, the 5e8-key float64 LogNormal(0,2) shard of one GPU
(seed 19, reference Rng + glibc libm, generated on the host). One step = one
sort of the config's arrays (C5: one array), each array by its own
lsort_cuda_sort call; every timed sort starts from a restored input (4 GB,
far above the 126 MB L2) and an untimed 256 MB L2-flush write, and is timed
with CUDA events on the sort's stream. `value` = keys sorted / summed device
time. Configs with several arrays (C2, C4) also report `overlapped`: the
arrays in one lsort_cuda_sort_many call.

`e2e`: the same sorts through the public API from pinned host memory (H2D and
D2H inside the timed region, wall clock around the synchronous call).

`cpu_baseline`: BASELINE.md section 3 on the box's host cores, on bounded
samples of the config (std::sort on one thread, __gnu_parallel::sort on all
cores, the AIPS2o port on all cores; mean of 10 runs).

N > 1 (torchrun): weak scaling, shard r of a world x n dataset per rank,
globally sorted across ranks; max over ranks of the device time.

--impl reference: the reference's CPU path (the oracle's C restatement of the
AIPS2o driver -- the reference ships no sort driver) on all host cores, on
this arm's config (whole arrays per step unless W + K steps would exceed
--ref-budget-s, then a bounded prefix sample, stated in the line).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (workload label, [(dist, seed)], n per array, key dtype)
    "c1": ("C1 uniform[0,1) f64 N=1e7 seed 42", [("uniform", 42)], 10_000_000, "f64"),
    "c2": ("C2 normal/lognormal(0,0.5)/exponential(2) f64 N=1e8 each seed 7",
           [("normal", 7), ("lognormal05", 7), ("exponential2", 7)], 100_000_000, "f64"),
    "c3": ("C3 mixture of 5 gaussians f64 N=2e8 seed 11", [("mixgauss", 11)], 200_000_000, "f64"),
    "c4": ("C4 rootdups/twodups/zipf(0.75) u64 N=1e8 seed 3",
           [("rootdups", 3), ("twodups", 3), ("zipf", 3)], 100_000_000, "u64"),
    "c5": ("C5 lognormal(0,2) f64 N=5e8 per GPU seed 19", [("lognormal2", 19)], 500_000_000, "f64"),
}
METRIC = "sorted keys/sec (Gkeys/s, float64) at 1/2/4/8 B200; % of HBM+NVLink roofline"


def passes(n_gpu: int) -> int:
    """BASELINE.md 2 / SURVEY 8(d): P = 1 + max(1, ceil(log_1024(N/16384)))."""
    import math
    return 1 + max(1, math.ceil(math.log(n_gpu / 16384, 1024)))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML
    polling thread (~2 ms period; nvidia-smi's 200 ms minimum period missed
    short regions), nvidia-smi as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None
        self.samples = []  # (sm_mhz, max_mhz, reason_mask)
        self._stop = None
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            # the visible device index maps to the NVML index through the UUID
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hi)
                    u = u.decode() if isinstance(u, bytes) else u
                    if uuid and uuid in u:
                        h = hi
                        break
            except Exception:
                pass
            self.h = h
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _poll(self):
        import time as _t
        nv, h = self.nv, self.h
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), self.max_mhz, int(rs)))
            except Exception:
                pass
            _t.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            import threading
            self._stop = threading.Event()
            self._thr = threading.Thread(target=self._poll, daemon=True)
            self._thr.start()
            return self
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0, set()
        if self.nv is not None:
            for f, m, rs in self.samples:
                sm.append(f)
                mx = max(mx, m)
                for nm, attr in self.REASONS:
                    if rs & int(getattr(self.nv, attr, 0)):
                        reasons.add(nm)
            src = "nvml"
        else:
            names = [r[0] for r in self.REASONS]
            for l in self.lines:
                f = [x.strip() for x in l.split(",")]
                try:
                    sm.append(float(f[0]))
                    mx = max(mx, float(f[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            src = "nvidia-smi"
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": src}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": src}


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# --------------------------------------------------------------------- CPU legs
def lscpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_arrays(cfg_name: str, n: int, first: int = 0, total: int | None = None):
    """Host inputs of a config (reference Rng + glibc libm, generated by the
    oracle's C restatement -- bit-identical to the library's lsort_gen_keys)."""
    from oracle import oracle as O
    label, dists, _, kind = CONFIGS[cfg_name]
    out = []
    for d, s in dists:
        if kind == "u64":  # shuffled datasets are generated whole; a prefix is a sample
            a = O.generate(d, total or n, s)[first:first + n].copy()
        else:
            a = O.generate(d, total or n, s, first=first, count=n)
        out.append(a)
    return out


def timed_port_sort(a: np.ndarray, threads: int) -> float:
    """One run of the AIPS2o CPU restatement (oracle, OpenMP) on a fresh copy; seconds."""
    from oracle import oracle as O
    b = a.copy()
    c = O.cfg(workers=threads)
    t0 = time.perf_counter()
    if b.dtype == np.float64:
        O.sort_doubles(b, c)
    else:
        O.sort_keys(b, c)
    return time.perf_counter() - t0


def cpu_baselines(cfg_name: str, runs: int = 10):
    """BASELINE.md section 3 on the box's host cores, each on a bounded sample of
    the config's first array, mean of `runs` runs:
    std::sort on one thread, __gnu_parallel::sort on all cores
    (the par_unseq stand-in) and the AIPS2o port (the oracle's
    C restatement of the reference driver, OpenMP, all cores)."""
    from oracle import oracle as O
    threads = O.lib().lso_max_threads()
    label, dists, n, kind = CONFIGS[cfg_name]
    samples = {"std_sort_1t": min(n, 10_000_000), "gnu_parallel_sort": min(n, 100_000_000),
               "aips2o_port": min(n, 20_000_000)}
    big = config_arrays(cfg_name, max(samples.values()), total=n)[0]
    keys = O.encode(big) if big.dtype == np.float64 else big
    res = {}
    for alg, m in samples.items():
        ts = []
        for _ in range(runs):
            if alg == "aips2o_port":
                ts.append(timed_port_sort(big[:m], threads))
                continue
            b = keys[:m].copy()
            t0 = time.perf_counter()
            if alg == "std_sort_1t":
                O.std_sort(b)
            else:
                O.parallel_sort(b, threads)
            ts.append(time.perf_counter() - t0)
        mean = float(np.mean(ts))
        res[alg] = {"value": m / mean / 1e9, "unit": "Gkeys/s", "keys": m, "runs": runs,
                    "threads": 1 if alg == "std_sort_1t" else threads, "mean_s": mean}
    return res, threads


def run_reference(args):
    """--impl reference: the reference's CPU path = the oracle's C restatement of
    the AIPS2o driver (the reference ships no sort driver, only its model layer;
    oracle/_ref holds that layer) on all host cores, on this arm's config. Each
    step sorts the whole config (every array, full size) from a fresh copy
    (untimed), unless W + K full steps would exceed the time budget, in which
    case each step sorts a bounded prefix sample (stated in `config`)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import oracle as O
    threads = O.lib().lso_max_threads()
    cfg_name = args.config
    label, dists, n, kind = CONFIGS[cfg_name]
    arrays = config_arrays(cfg_name, n)
    # first warm-up step on the full config decides whether full steps fit the budget
    t_full = sum(timed_port_sort(a, threads) for a in arrays)
    m = n
    if t_full * (args.warmup + args.steps) > args.ref_budget_s:
        m = max(1_000_000, int(n * args.ref_budget_s / (t_full * (args.warmup + args.steps))))
        arrays = [a[:m].copy() for a in arrays]
    ts = []
    for step in range(args.warmup - 1 + args.steps):
        t = sum(timed_port_sort(a, threads) for a in arrays)
        if step >= args.warmup - 1:
            ts.append(t)
    t = float(np.mean(ts))
    v = len(arrays) * m / t / 1e9
    sample = ("full config per step" if m == n else f"{m} keys (prefix) of each of {len(arrays)} arrays per step; "
              f"a full-config step took {t_full:.1f} s")
    line = {"metric": METRIC, "value": v, "unit": "Gkeys/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": kind, "data": DATA, "impl": "reference",
            "config": config_dict(cfg_name, world=1),
            "cpu_baseline": {"value": v, "unit": "Gkeys/s", "cores": threads, "kind": "port",
                             "sample": sample, "cpu_model": lscpu_model()},
            "e2e": {"value": v, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if m != n:
        line["config"]["reference_sample_keys_per_array"] = m
    print(json.dumps(line), flush=True)


DATA = "synthetic (reference Rng splitmix64 + glibc libm on host; BASELINE.json seeds)"


def config_dict(cfg_name: str, world: int, n: int | None = None) -> dict:
    label, dists, n0, kind = CONFIGS[cfg_name]
    return {"workload": label, "keys_per_array_per_gpu": n or n0, "arrays": len(dists),
            "l2": "inputs (>= 80 MB, > 126 MB L2 from C2 up) restored + 256 MB L2-flush write before every timed sort",
            "parallelism": f"dp{world}" if world > 1 else "single-gpu"}


def traffic_profile(cfg_name: str):
    """Measured DRAM bytes per key per phase for this config (ncu counters over
    one sort of each config array, tools/phase_traffic.py) -- or None."""
    path = os.path.join(ROOT, "profiles", f"r2_traffic_{cfg_name}.json")
    try:
        with open(path) as f:
            return json.load(f), os.path.relpath(path, ROOT)
    except (OSError, ValueError):
        return None, None


# --------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import paper_2307_08637_b200 as L

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist_mode = world > 1 or args.dist
    if dist_mode:
        return run_dist(args)
    label, dists, n, kind = CONFIGS[args.config]
    if args.keys:
        n = args.keys
    dev = torch.device("cuda", local)

    # ---- inputs (host generation, reference Rng), pristine device copies
    hosts = config_arrays(args.config, n)
    pristine = [torch.from_numpy(h.view(np.int64) if h.dtype == np.uint64 else h).to(dev) for h in hosts]
    work = [torch.empty_like(p) for p in pristine]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ctx = L.Context(local)
    cfg = L.SortConfig()
    cfg_phase = L.SortConfig(flags=L._native.FLAG_PHASE_TIMING)

    def restore(i):
        work[i].copy_(pristine[i])
        flush.fill_(1)
        torch.cuda.synchronize()

    api_ms = [0.0]

    def one_sort(i, c=cfg):
        """untimed restore + L2 flush, then the event-timed sort of array i (ms, stats).
        The time is the library's own CUDA events on its stream around the sort's
        device work (lsort_stats.ms_total: first to last enqueued command, host gaps
        between levels included); the torch events around the Python call (which
        also hold the ctypes call, argument checks and the final host sync, ~0.1 ms)
        are reported beside it as api_ms_per_step."""
        restore(i)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        stats = ctx.sort(work[i], c)
        e1.record(st)
        torch.cuda.synchronize()
        api_ms[0] += e0.elapsed_time(e1)
        return stats["ms_total"], stats

    for _ in range(args.warmup):
        for i in range(len(work)):
            one_sort(i)
    for i in range(len(work)):  # correctness spot check on a warm-up output (untimed)
        one_sort(i)
        ok, fv, _ = ctx.verify(work[i])
        if not ok:
            raise SystemExit(f"output {i} not sorted at {fv}")
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    total_ms, launches, levels = 0.0, 0, 0
    api_ms[0] = 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            for i in range(len(work)):
                ms, stats = one_sort(i)
                total_ms += ms
                launches += stats.get("kernel_launches", 0)
                levels += stats.get("levels", 0)
    clocks = clk.summary()
    nsorts = args.steps * len(work)
    ms_per_step = total_ms / args.steps
    api_ms_per_step = api_ms[0] / args.steps
    keys_per_step = len(work) * n
    value = keys_per_step / (ms_per_step * 1e-3) / 1e9

    # ---- per-phase breakdown: an extra untimed pass with per-phase events
    phases = {k: 0.0 for k in PHASES}
    part_keys = base_keys = direct_keys = 0
    for i in range(len(work)):
        _, st_ph = one_sort(i, cfg_phase)
        for k in PHASES:
            phases[k] += st_ph.get(k, 0.0) / len(work)
        part_keys += st_ph["partitioned_keys"] / len(work)
        base_keys += st_ph["base_case_keys"] / len(work)
        direct_keys += st_ph.get("direct_keys", 0) / len(work)
    # algorithmic bytes per launch of each phase: the
    # scatter moves every partitioned key once (8 B read + 8 B write; the padded
    # one-pass level 0 counts here), the base case reads + writes each
    # base-case key once, the classify reads each key of a two-pass level once
    alg = {"ms_scatter": 16.0 * part_keys, "ms_base": 16.0 * base_keys,
           "ms_classify": 8.0 * (part_keys - direct_keys)}
    dom = max(alg, key=lambda k: phases[k])
    achieved = alg[dom] / (phases[dom] * 1e-3) / 1e9 if phases[dom] > 0 else 0.0
    tj, tsrc = traffic_profile(args.config)
    traffic = None
    if tj is not None:
        ph = {"ms_scatter": "scatter", "ms_base": "base", "ms_classify": "classify"}[dom]
        traffic = tj["phases"][ph]["dram_bytes_per_key"] * n
    P = passes(n)
    t_roof_ms = 16.0 * P * n / (hbm * 1e9) * 1e3 * len(work)
    line = {
        "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": kind, "data": DATA,
        "config": config_dict(args.config, 1, n),
        "roofline": {"bound": "hbm", "kernel": PHASE_KERNEL[dom], "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "traffic_source": tsrc, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg[dom],
                     "note": "phase = all launches of that kernel in one sort (per-phase CUDA events)"},
        "sort_roofline": {"passes": P, "bytes_per_key": 16 * P, "t_roof_ms_per_step": t_roof_ms,
                          "frac": t_roof_ms / ms_per_step, "hbm_gbs": hbm},
        "phases_ms_per_sort": phases,
        "api_ms_per_step": api_ms_per_step,
        "schedule": "one sort at a time (each array of the config sorted by its own lsort_cuda_sort call)",
        "levels_per_sort": levels / nsorts,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if len(work) > 1:  # the config's arrays in flight together (lsort_cuda_sort_many), beside the headline
        ms_b = []
        for r in range(6):  # (rep 0 warms the sub-contexts: their workspaces grow on first use)
            for i in range(len(work)):
                work[i].copy_(pristine[i])
            flush.fill_(1)
            torch.cuda.synchronize()
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.sort_batch(work, cfg)
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                ms_b.append(e0.elapsed_time(e1))
        for i in range(len(work)):
            ok, fv, _ = ctx.verify(work[i])
            if not ok:
                raise SystemExit(f"sort_many output {i} not sorted at {fv}")
        mb = float(np.median(ms_b))
        line["overlapped"] = {"value": keys_per_step / (mb * 1e-3) / 1e9, "unit": "Gkeys/s", "ms_per_step": mb,
                              "schedule": "the config's arrays in one lsort_cuda_sort_many call (3 sorts in flight)"}
    # ---- e2e through the public API from pinned host memory (H2D + D2H inside)
    if args.e2e_steps > 0:
        del pristine, work
        torch.cuda.empty_cache()
        pins = [torch.empty(n, dtype=torch.float64 if h.dtype == np.float64 else torch.int64, pin_memory=True)
                for h in hosts]
        arrs = [p.numpy() if h.dtype == np.float64 else p.numpy().view(np.uint64) for p, h in zip(pins, hosts)]
        e2e_t = []
        for step in range(args.e2e_steps + 1):
            for a, h in zip(arrs, hosts):
                a[...] = h
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if len(arrs) == 1:
                ctx.sort(arrs[0], cfg)  # lsort_cuda_sort, LSORT_MEM_HOST
            else:
                ctx.sort_batch(arrs, cfg)  # lsort_cuda_sort_batch: copies pipelined against the sorts
            dt = time.perf_counter() - t0
            if step > 0:
                e2e_t.append(dt)
        for a in arrs:  # the end-to-end result is checked, not just timed
            k = O_encode(a) if a.dtype == np.float64 else a
            if not np.all(k[1:] >= k[:-1]):
                raise RuntimeError("e2e sort produced unsorted output")
        e2e_ms = float(np.mean(e2e_t)) * 1e3
        line["e2e"] = {"value": keys_per_step / (e2e_ms * 1e-3) / 1e9, "unit": "Gkeys/s",
                       "h2d_bytes_per_step": 8 * n * len(arrs), "d2h_bytes_per_step": 8 * n * len(arrs),
                       "ms_per_step": e2e_ms,
                       "api": "lsort_cuda_sort (LSORT_MEM_HOST)" if len(arrs) == 1 else "lsort_cuda_sort_batch"}
    else:
        line["e2e"] = None
    if not args.no_cpu:
        res, threads = cpu_baselines(args.config, args.cpu_runs)
        port = res["aips2o_port"]
        line["cpu_baseline"] = {"value": port["value"], "unit": "Gkeys/s", "cores": threads, "kind": "port",
                                "sample": f"{port['keys']} keys of the config's first array, mean of {port['runs']}",
                                "cpu_model": lscpu_model(), "algorithms": res}
    print(json.dumps(line), flush=True)


def O_encode(a):
    from oracle import oracle as O
    return O.encode(a)


PHASES = ("ms_models", "ms_classify", "ms_scatter", "ms_base", "ms_fill")
PHASE_KERNEL = {"ms_scatter": "k_direct (level 0) + k_scatter", "ms_base": "k_base_reg/k_base_smem", "ms_classify": "k_hist"}


def run_dist(args):
    """N > 1 (torchrun, one process per GPU): weak scaling, shard r of the
    config (keys [r n, (r+1) n) of a world x n dataset), globally sorted
    across ranks by the multi-GPU driver (lsort_cuda_sort_dist through
    paper_2307_08637_b200.dist.DistContext: global model, rank cuts, the
    exchange fused into the level-0 scatter over NVLink, local sort).
    Max over ranks of the CUDA-event time of each sort."""
    import torch
    import torch.distributed as tdist
    import paper_2307_08637_b200 as L
    from paper_2307_08637_b200.dist import DistContext
    rank, world, local = env_rank()
    for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533")):
        os.environ.setdefault(k, v)  # --dist without torchrun: a one-rank group
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    label, dists, n, kind = CONFIGS[args.config]
    if args.keys:
        n = args.keys
    dev = torch.device("cuda", local)
    hosts = config_arrays(args.config, n, first=rank * n, total=world * n) if kind == "f64" else \
        config_arrays(args.config, n)
    pristine = [torch.from_numpy(h.view(np.int64) if h.dtype == np.uint64 else h).to(dev) for h in hosts]
    work = [torch.empty_like(p) for p in pristine]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ctx = L.Context(local)  # (verify)
    dc = DistContext(local)  # one rank of the multi-GPU driver (the library owns its NCCL communicator)
    cfg = L.SortConfig()

    def one_sort(i):
        work[i].copy_(pristine[i])
        flush.fill_(1)
        torch.cuda.synchronize()
        tdist.barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        out, stats = dc.sort(work[i], cfg)
        e1.record(st)
        torch.cuda.synchronize()
        tdist.barrier()
        return e0.elapsed_time(e1), stats, out

    for _ in range(args.warmup):
        for i in range(len(work)):
            one_sort(i)
    for i in range(len(work)):
        _, _, out = one_sort(i)
        ok, fv, _ = ctx.verify(out)
        if not ok:
            raise SystemExit(f"rank {rank}: output {i} not sorted at {fv}")
    total_ms, launches = 0.0, 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            for i in range(len(work)):
                ms, stats, _ = one_sort(i)
                total_ms += ms
                launches += stats.get("kernel_launches", 0)
    clocks = clk.summary()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    keys_per_step = len(work) * n * world
    value = keys_per_step / (ms_per_step * 1e-3) / 1e9
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    P = passes(n)
    t_roof_ms = (16.0 * P * n / (hbm * 1e9) + 8.0 * n * (world - 1) / world / 900e9) * 1e3 * len(work)
    line = {"metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": kind, "data": DATA, "config": config_dict(args.config, world, n),
            "sort_roofline": {"passes": P, "bytes_per_key": 16 * P, "nvlink_bytes_per_key": 8 * (world - 1) / world,
                              "t_roof_ms_per_step": t_roof_ms, "frac": t_roof_ms / ms_per_step, "hbm_gbs": hbm},
            "gpu_launches": int(launches), "clocks": clocks, "e2e": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--keys", type=int, default=0, help="override keys per array (testing)")
    ap.add_argument("--cpu-runs", type=int, default=10)
    ap.add_argument("--ref-budget-s", type=float, default=240.0, help="reference arm: time budget of W + K steps")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true", help="force the distributed path (also at 1 rank)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: W < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
