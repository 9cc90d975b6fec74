#!/usr/bin/env python
"""Benchmark: sorted keys/s of the B200 LearnedSort (AIPS2o) on BASELINE.json's configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Default workload (N=1) = BASELINE.json configs[1] ("C2"): N = 1e8 float64
keys per array, three arrays -- Normal(0,1), LogNormal(0,0.5), Exponential(2),
i.i.d. from seed 7 (reference Rng, glibc libm, generated on the host). One
step = sorting the three arrays (3e8 keys). Inputs (800 MB each) are larger
than the 126 MB L2, restored from pristine device copies before every step
(untimed), followed by an untimed 256 MB L2-flush write. Each sort is
bracketed by barrier + synchronize and timed with CUDA events on the sort's
stream; `value` = keys sorted / summed device time (max over ranks).

N > 1 (torchrun): weak scaling, 1e8 keys of each C2 distribution per rank,
globally sorted across ranks (RMI splitters + NCCL all-to-all, see
paper_2307_08637_b200/dist.py).

--impl reference: the reference's CPU path (oracle/ C restatement of the
AIPS2o driver; the reference ships no sort driver) on the host cores, on a
bounded sample of the same workload per step.
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
def cpu_sort_rate(cfg_name: str, sample_n: int, runs: int):
    """Oracle AIPS2o restatement (OpenMP, all host threads) on `sample_n` keys
    of each config distribution; returns (Mkeys/s list per run, threads)."""
    from oracle import oracle as O
    label, dists, n, kind = CONFIGS[cfg_name]
    threads = os.cpu_count() or 1
    arrays = [O.generate(d, n if kind == "u64" else sample_n, s) for d, s in dists]
    if kind == "u64":  # shuffled datasets are generated whole; take a prefix
        arrays = [a[:sample_n].copy() for a in arrays]
    rates = []
    c = O.cfg(workers=threads)
    for _ in range(runs):
        t = 0.0
        for a in arrays:
            b = a.copy()
            t0 = time.perf_counter()
            if kind == "f64":
                O.sort_doubles(b, c)
            else:
                O.sort_keys(b, c)
            t += time.perf_counter() - t0
        rates.append(len(arrays) * sample_n / t / 1e9)
    return rates, threads


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    cfg_name = args.config
    label, dists, n, kind = CONFIGS[cfg_name]
    sample_n = min(n, args.cpu_sample)
    rates, threads = cpu_sort_rate(cfg_name, sample_n, args.warmup + args.steps)
    timed = rates[args.warmup:]
    v = float(np.mean(timed))
    ms = len(dists) * sample_n / (v * 1e9) * 1e3
    line = {"metric": METRIC, "value": v, "unit": "Gkeys/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": kind, "data": "synthetic (reference Rng, host)",
            "impl": "reference",
            "config": {"workload": label, "sample_keys_per_array": sample_n, "arrays": len(dists)},
            "cpu_baseline": {"value": v, "unit": "Gkeys/s", "cores": threads, "kind": "port",
                             "sample": f"{sample_n} keys x {len(dists)} arrays per step"},
            "e2e": {"value": v, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import paper_2307_08637_b200 as L

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist_mode = world > 1 or args.dist
    if dist_mode:
        import torch.distributed as tdist
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533")):
            os.environ.setdefault(k, v)  # --dist without torchrun: a one-rank group
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    label, dists, n, kind = CONFIGS[args.config]
    if args.keys:
        n = args.keys
    f64 = kind == "f64"
    dev = torch.device("cuda", local)

    # ---- inputs (host generation, reference Rng; shard r of a world*n dataset)
    pristine = []
    for d, s in dists:
        if dist_mode and kind == "f64":
            h = L.generate(d, world * n, s, first=rank * n, count=n)
        else:
            h = L.generate(d, n, s)
        t = torch.from_numpy(h.view(np.int64) if h.dtype == np.uint64 else h).to(dev)
        pristine.append(t)
    work = [torch.empty_like(p) for p in pristine]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ctx = L.Context(local)
    # timed sorts run without per-phase events (those force a host sync per
    # level); an extra untimed pass with LSORT_FLAG_PHASE_TIMING feeds the
    # per-phase roofline. The distributed path keeps them (per-rank phases).
    cfg_phase = L.SortConfig(flags=L._native.FLAG_PHASE_TIMING)
    cfg = cfg_phase if dist_mode else L.SortConfig()
    if dist_mode:
        from paper_2307_08637_b200.dist import DistSorter
        sorter = DistSorter(ctx, cfg)

    def barrier():
        if dist_mode:
            import torch.distributed as tdist
            tdist.barrier()

    def one_sort(i):
        """restore + flush (untimed), then timed sort of array i; returns (ms, stats)."""
        work[i].copy_(pristine[i])
        flush.fill_(1)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        if dist_mode:
            out, stats = sorter.sort(work[i])
        else:
            stats = ctx.sort(work[i], cfg)
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        return ms, stats, (out if dist_mode else work[i])

    def batch_step():
        """restore + flush (untimed), then ONE timed lsort_cuda_sort_many call over
        all arrays of the config (up to three sorts in flight on separate contexts)."""
        for i in range(len(work)):
            work[i].copy_(pristine[i])
        flush.fill_(1)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        stats = ctx.sort_batch(work, cfg)
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), stats

    use_batch = not dist_mode and len(work) > 1 and not args.sequential
    for _ in range(args.warmup):
        for i in range(len(work)):
            one_sort(i)
        if use_batch:
            batch_step()
    # correctness spot check on the last warm-up output (untimed)
    for i in range(len(work)):
        _, _, res = one_sort(i)
        ok, fv, _ = ctx.verify(res)
        if not ok:
            raise SystemExit(f"rank {rank}: output {i} not sorted at {fv}")
    peaks, peak_src = measured_peaks()
    total_ms = 0.0
    agg = {}
    launches = 0
    seq_ms = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if use_batch:
                ms, stats = batch_step()
                total_ms += ms
                launches += stats.get("kernel_launches", 0)
                for k, v in stats.items():
                    if isinstance(v, (int, float)):
                        agg[k] = agg.get(k, 0) + v
                continue
            for i in range(len(work)):
                ms, stats, _ = one_sort(i)
                total_ms += ms
                if dist_mode:
                    stats = dict(stats.get("local") or {})
                launches += stats.get("kernel_launches", 0)
                for k, v in stats.items():
                    if isinstance(v, (int, float)):
                        agg[k] = agg.get(k, 0) + v
    clocks = clk.summary()
    if use_batch:  # the same arrays one sort at a time (reported beside the headline)
        for _ in range(2):
            seq_ms = sum(one_sort(i)[0] for i in range(len(work)))
        for i in range(len(work)):  # the batch output is checked too
            work[i].copy_(pristine[i])
        ctx.sort_batch(work, cfg)
        for i in range(len(work)):
            ok, fv, _ = ctx.verify(work[i])
            if not ok:
                raise SystemExit(f"batch output {i} not sorted at {fv}")
    if not dist_mode:  # phase breakdown (untimed)
        for k in ("ms_models", "ms_classify", "ms_scatter", "ms_base", "ms_fill"):
            agg[k] = 0.0
        for i in range(len(work)):
            work[i].copy_(pristine[i])
            st_ph = ctx.sort(work[i], cfg_phase)
            for k in ("ms_models", "ms_classify", "ms_scatter", "ms_base", "ms_fill"):
                agg[k] += st_ph.get(k, 0.0) * args.steps  # scaled like the timed aggregate
    keys_per_step = len(work) * n * (world if dist_mode else 1)
    if dist_mode:
        import torch.distributed as tdist
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = keys_per_step / (ms_per_step * 1e-3) / 1e9  # Gkeys/s whole job

    # ---- roofline: dominant kernel (by measured phase share) and whole sort
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    nsteps_arrays = args.steps * len(work)
    phases = {k: agg.get(k, 0.0) / nsteps_arrays for k in
              ("ms_models", "ms_classify", "ms_scatter", "ms_base", "ms_fill")}
    # algorithmic bytes per launch: scatter moves every partitioned key once
    # (8 B read + 8 B write); base case reads + writes each base-case key once;
    # classify reads each partitioned key once (8 B).
    part_keys = agg.get("partitioned_keys", 0) / nsteps_arrays
    base_keys = agg.get("base_case_keys", 0) / nsteps_arrays
    alg = {"ms_scatter": 16.0 * part_keys, "ms_base": 16.0 * base_keys, "ms_classify": 8.0 * part_keys}
    dom = max(alg, key=lambda k: phases[k])
    achieved = alg[dom] / (phases[dom] * 1e-3) / 1e9 if phases[dom] > 0 else 0.0
    names = {"ms_scatter": "k_scatter", "ms_base": "k_base", "ms_classify": "k_classify_hist"}
    # measured DRAM bytes of the same phase (ncu counters, profiles/r1_kernel_traffic.json),
    # scaled to this run's keys per sort
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "r1_kernel_traffic.json")))
        ph = {"ms_scatter": "scatter", "ms_base": "base", "ms_classify": "classify"}[dom]
        traffic = tj["phases"][ph]["dram_bytes_per_key"] * n
    except (OSError, KeyError, ValueError):
        traffic = None
    nper = n
    P = passes(nper)
    t_roof_ms = 16.0 * P * nper / (hbm * 1e9) * 1e3 * len(work)
    if dist_mode:
        t_roof_ms += 8.0 * nper * (world - 1) / world / 770e9 * 1e3 * len(work)
    line = {
        "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": kind,
        "data": "synthetic (reference Rng splitmix64 + glibc libm on host; BASELINE.json seeds)",
        "config": {"workload": label, "keys_per_array_per_gpu": n, "arrays": len(work),
                   "l2": "inputs (>=80 MB) restored + 256 MB L2 flush before every timed sort",
                   "parallelism": f"dp{world}" if dist_mode else "single-gpu"},
        "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "traffic_source": "profiles/r1_kernel_traffic.json (ncu DRAM counters, C2 normal 1e8)",
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg[dom]},
        "sort_roofline": {"passes": P, "bytes_per_key": 16 * P, "t_roof_ms_per_step": t_roof_ms,
                          "frac": t_roof_ms / ms_per_step, "hbm_gbs": hbm},
        "phases_ms_per_sort": phases,
        "schedule": ("the config's arrays in one lsort_cuda_sort_many call (up to 3 sorts in flight)"
                     if use_batch else "one sort at a time"),
        "sequential": ({"value": keys_per_step / (seq_ms * 1e-3) / 1e9, "unit": "Gkeys/s", "ms_per_step": seq_ms}
                       if seq_ms else None),
        "levels_per_sort": agg.get("levels", 0) / nsteps_arrays,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    # ---- e2e through the public API with pinned host buffers (H2D + D2H inside)
    if not dist_mode and args.e2e_steps > 0:
        hosts = [torch.empty(n, dtype=p.dtype, pin_memory=True) for p in pristine]
        src = [p.cpu() for p in pristine]
        # the public batch entry point (lsort_cuda_sort_batch): one call sorts
        # the config's arrays from pinned host memory, copies in / out
        # pipelined against the sorts on two copy streams
        e2e_t = 0.0
        for step in range(args.e2e_steps + 1):
            arrs = []
            for i in range(len(hosts)):
                hosts[i].copy_(src[i])
                arrs.append(hosts[i].numpy())
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.sort_batch(arrs, cfg)
            dt = time.perf_counter() - t0
            if step > 0:
                e2e_t += dt
        for i in range(len(hosts)):  # the end-to-end result is checked, not just timed
            ok, _, _ = ctx.verify(torch.from_numpy(hosts[i].numpy()).cuda())
            if not ok:
                raise RuntimeError("e2e sort produced unsorted output")
        e2e_ms = e2e_t / max(1, args.e2e_steps) * 1e3
        line["e2e"] = {"value": len(hosts) * n / (e2e_ms * 1e-3) / 1e9, "unit": "Gkeys/s",
                       "h2d_bytes_per_step": 8 * n * len(hosts), "d2h_bytes_per_step": 8 * n * len(hosts),
                       "ms_per_step": e2e_ms}
    elif dist_mode and args.e2e_steps > 0:
        # the distributed public API end to end: every rank copies its shard in
        # from pinned host memory, the global sort runs (RMI splitters + NCCL
        # all-to-all + local sort), and the rank's output range is read back to
        # pinned host memory -- CUDA events around all of it, max over ranks
        import torch.distributed as tdist
        hosts = [p.cpu().pin_memory() for p in pristine]
        # result buffers pinned up front (a rank receives ~n keys; larger ranges
        # get a fresh buffer); copies in / out on their own streams, pipelined
        # against the sorts: array i+1 streams in while array i sorts
        cap = int(1.5 * n) + 4096
        outs = [torch.empty(cap, dtype=torch.int64, pin_memory=True) for _ in pristine]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        e2e_ms, d2h = 0.0, 0
        for step in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            barrier()
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s_in.wait_stream(st)
            ev_in = []
            for i in range(len(hosts)):
                with torch.cuda.stream(s_in):
                    work[i].copy_(hosts[i], non_blocking=True)
                    ev_in.append(torch.cuda.Event())
                    ev_in[-1].record(s_in)
            step_d2h, keep = 0, []
            for i in range(len(hosts)):
                st.wait_event(ev_in[i])
                out, _ = sorter.sort(work[i])
                o64 = out.view(torch.int64)
                dst = outs[i] if o64.numel() <= cap else torch.empty(o64.numel(), dtype=torch.int64, pin_memory=True)
                s_out.wait_stream(st)
                with torch.cuda.stream(s_out):
                    dst[: o64.numel()].copy_(o64, non_blocking=True)
                keep.append(out)
                step_d2h += o64.numel() * 8
            st.wait_stream(s_out)
            e1.record(st)
            torch.cuda.synchronize()
            if step > 0:
                e2e_ms += e0.elapsed_time(e1)
                d2h += step_d2h
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t.item()) / max(1, args.e2e_steps)
        line["e2e"] = {"value": keys_per_step / (e2e_ms * 1e-3) / 1e9, "unit": "Gkeys/s",
                       "h2d_bytes_per_step": 8 * n * len(hosts),
                       "d2h_bytes_per_step": int(d2h / max(1, args.e2e_steps)),
                       "ms_per_step": e2e_ms, "per_rank_bytes": True}
    else:
        line["e2e"] = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample_n = min(n, args.cpu_sample)
        rates, threads = cpu_sort_rate(args.config, sample_n, 2)
        line["cpu_baseline"] = {"value": float(np.mean(rates)), "unit": "Gkeys/s", "cores": threads,
                                "kind": "port",
                                "sample": f"{sample_n} keys of each of {len(work)} config arrays, 2 runs"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_mode:
        import torch.distributed as tdist
        tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--keys", type=int, default=0, help="override keys per array (testing)")
    ap.add_argument("--cpu-sample", type=int, default=10_000_000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true", help="force the distributed path (also at 1 rank)")
    ap.add_argument("--sequential", action="store_true", help="time the arrays one sort at a time")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: W < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
