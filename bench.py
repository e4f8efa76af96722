#!/usr/bin/env python3
"""Benchmark: full PF-SMC particle-steps/s of the per-observation update
(BASELINE.json metric) on BASELINE config 2 — Lotka-Volterra, N = 2^20
particles per GPU, FP64, h = 0.1 (one LMM step per observation), a = 0.98,
synthetic RK4 observations.

One bench "step" = one pf_step (filter.cpp:292-394) over the whole resident
ensemble for the next observation. Timing: per-step CUDA events on the
sampler's stream, W >= 3 warm-up steps, the L2 flushed (256 MiB write)
between timed steps outside the events; max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: the unmodified C++ pf_step, Backend::parallel(all host
threads)) on the same workload, each step a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec (full PF-SMC step)"
UNIT = "particle-steps/s"
N_PER_GPU = 1 << 20
T_OBS = 1000
# Algorithmic bytes per particle, F = d + p + 1.
D, P = 2, 2
F = D + P + 1
STEP_BYTES = 24 * F + 56                     # whole step, minimal fused pipeline
R = D + P                                     # record doubles (x, theta_u)
KERNEL_BYTES = {                              # per particle per launch
    "k_predict": 8 * R + 8 + 8 + 8,           # record + lw in; ll_bar + lg out
    "k_scan_pieces": 8 + 8,                   # lg in; g out
    "k_scan_cdf": 8 + 8 + 2,                  # g in; cdf + local guide out
    "k_scan_fused": 8 + 8 + 2,                # lg in; cdf + search tables out (single-pass scan)
    "k_serve": 8 * R + 8 + 8 * (R + 2) + 4,   # ancestor record + ll_bar gathered; payload + anc out
    "k_update": 8 * (R + 2) + 8 * R + 8,      # payload in; record + lw out
}


# FP64 flops the device executes per chain Newton iteration (banded path,
# lmm.cuh band_solve + ChainModel::rhs_jac_band, counting FMA as 2 and a
# division as 1): rhs + band 13 div + 7 add + 7 mul (flux), 6x(2 mul + sub + sub)
# + 2 mul + sub (o), 6 mul (den^2), 7x(mul + mul + sub) (jd) ~ 80; residual 3x8;
# band: 2 mul + add per diagonal and sub-diagonal entry ~ 45, 7 reciprocals,
# 7x(mul + mul + sub) forward, 8 divisions back; update + norms 8x(sub + 2 abs)
EXEC_FLOPS_PER_NEWTON_CHAIN = 80 + 24 + 45 + 7 + 21 + 8 + 24


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


_POLLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
bus = sys.argv[1]
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(bus)
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
        nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
print("ready", flush=True)
while True:
    t = time.monotonic()
    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    try:
        r = fn(h)
    except Exception:
        r = 0
    print(f"{t:.6f},{sm},{mx}," + ",".join("1" if r & b else "0" for b in bits), flush=True)
    time.sleep(float(sys.argv[3]))
"""


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    A separate process polls NVML (nvidia_ml_py) every ~1 ms and prints
    CLOCK_MONOTONIC-stamped samples (no GIL contention with the timing loop);
    the summary keeps the samples inside [enter, exit] of the timed region.
    The poller is started and confirmed ready before the region begins.
    """

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, period_s: float = 0.001):
        self.index = index
        self.period = period_s
        self.rows = []          # (t, sm_mhz, max_mhz, [reason names])
        self.proc = None
        self.err = None
        self.t0 = self.t1 = None

    def _bus_id(self):
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            return f"{getattr(pr, 'pci_domain_id', 0):08x}:{pr.pci_bus_id:02x}:{getattr(pr, 'pci_device_id', 0):02x}.0"
        except Exception:  # noqa: BLE001
            return ""

    def _read(self):
        for line in self.proc.stdout:
            f = line.strip().split(",")
            if len(f) < 7:
                continue
            try:
                self.rows.append((float(f[0]), float(f[1]), float(f[2]),
                                  [n for n, v in zip(self.NAMES, f[3:7]) if v == "1"]))
            except ValueError:
                pass

    def __enter__(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _POLLER, self._bus_id(), str(self.index),
                                          str(self.period)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                         text=True)
            first = self.proc.stdout.readline()  # blocks until the poller has NVML up
            if not first.startswith("ready"):
                self.err = (first + self.proc.stderr.read())[-200:]
                self.proc = None
            else:
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
                time.sleep(0.005)
        except Exception as e:  # noqa: BLE001
            self.err, self.proc = repr(e)[:200], None
        self.t0 = time.monotonic()
        return self

    def __exit__(self, *a):
        self.t1 = time.monotonic()
        if self.proc:
            time.sleep(0.003)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        inside = [r for r in self.rows if self.t0 is not None and self.t0 <= r[0] <= self.t1]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err,
                    "samples_total": len(self.rows)}
        sm = [r[1] for r in inside]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[2] for r in inside),
                "reasons": sorted({n for r in inside for n in r[3]}), "samples": len(inside),
                "region_ms": (self.t1 - self.t0) * 1e3, "source": "nvml poller process"}


def _issue_floor(prof, avg_ms, clocks):
    wi = prof.get("warp_inst_per_launch")
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz")
    if not wi or not mhz:
        return {}
    try:
        import torch
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    except Exception:  # noqa: BLE001
        sms = 148
    floor_us = wi / (sms * 4 * mhz * 1e6) * 1e6
    return {"ncu_warp_inst_per_launch": wi, "issue_floor_us": floor_us,
            "frac_of_issue_floor": floor_us / (avg_ms * 1e3)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference(n, steps, seconds_cap, workers, prob, use_ref=True, warmup=0):
    """Times the reference (oracle/_ref) or the C port on a bounded sample,
    after `warmup` untimed steps of the same sequence."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ctypes import REF_SO, Oracle, Reference, StepConfig
    kind = "reference" if (use_ref and os.path.exists(REF_SO)) else "port"
    O = Oracle()
    sc = StepConfig(model="lv", family=prob.cfg.family, order=prob.cfg.order, h=0.1, a=0.98,
                    seed=prob.cfg.seed, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, prob.cfg.seed, **prob.prior)
    done, secs = 0, 0.0
    tp = 0.0
    for j in range(1, warmup + 1):  # untimed warm-up steps (same observation sequence)
        t1 = prob.times[j - 1]
        if kind == "reference":
            Reference().time_steps(sc, ens, prob.ys[j - 1:j], [t1], j, tp, workers)
        else:
            O.pf_step(sc, ens, prob.ys[j - 1], j, tp, t1)
        tp = t1
    while done < steps and (secs < seconds_cap or done < 1):
        j = warmup + done + 1
        t1 = prob.times[j - 1]
        if kind == "reference":
            secs += Reference().time_steps(sc, ens, prob.ys[j - 1:j], [t1], j, tp, workers)
        else:
            t0 = time.perf_counter()
            O.pf_step(sc, ens, prob.ys[j - 1], j, tp, t1)
            secs += time.perf_counter() - t0
        tp = t1
        done += 1
    return {"value": n * done / secs, "unit": UNIT, "cores": workers if kind == "reference" else 1,
            "kind": kind, "steps": done, "seconds": secs,
            "sample": f"LV N={n}, observations {warmup + 1}..{warmup + done} (after {warmup} untimed), "
                      + (f"reference pf_step Backend::parallel({workers})" if kind == "reference"
                         else "C restatement, 1 thread")}


def _lv_config(world, n):
    """The headline workload's config dict, identical in both arms."""
    return {"workload": "BASELINE config 2: Lotka-Volterra PF-SMC", "particles_per_gpu": n,
            "global_particles": n * world, "d": D, "p": P, "h": 0.1, "shrink_a": 0.98,
            "integrator": "am2 (reference semantics: m=1 => AM1 corrector, AB1 predictor)",
            "l2": "flushed between timed steps (256 MiB write, outside the events)",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_sequential(prob, n=1 << 16):
    """The reference pf_step with Backend::sequential() (exec.hpp:47-62) on one
    observation at n particles (its throughput is flat in N)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_ctypes import REF_SO, Oracle, Reference, StepConfig
        if not os.path.exists(REF_SO):
            return None
        sc = StepConfig(model="lv", family=prob.cfg.family, order=prob.cfg.order, h=0.1, a=0.98,
                        seed=prob.cfg.seed, obs_idx=(0, 1), sigma=0.05)
        ens = Oracle().init_uniform("lv", n, prob.cfg.seed, **prob.prior)
        secs = Reference().time_steps(sc, ens, prob.ys[0:2], list(prob.times[0:2]), 1, 0.0, 0)
        return {"value": 2 * n / secs, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"LV N={n}, observations 1..2, reference pf_step Backend::sequential()"}
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)[:200]}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    from paper_1411_1702_b200 import problems
    workers = len(os.sched_getaffinity(0))
    prob = problems.lotka_volterra(particles=N_PER_GPU, T=max(args.steps + args.warmup, 4), seed=1)
    # each step: one reference pf_step at the full N = 2^20 (bounded: <= 30 s total)
    # warm-up steps are bounded too (at most 3: each is ~1 s of 16 host threads at N = 2^20).
    # Exactly K timed steps; beyond 32 of them each step is a smaller sample of the
    # ensemble (the reference's throughput is flat in N), so the run
    # stays within a few minutes.
    w = max(args.warmup, 3)  # the same W as the GPU arm (bench.py forces W >= 3 there too)
    n_ref = N_PER_GPU
    while args.steps * n_ref > 32 * N_PER_GPU and n_ref > (1 << 14):
        n_ref //= 2
    cb = cpu_reference(n_ref, args.steps, 240.0, workers, prob, warmup=w)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": cb["steps"],
            "warmup": w, "ms_per_step": 1e3 * cb["seconds"] / cb["steps"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded RK4 LV)",
            "impl": "reference",
            "config": _lv_config(args.gpus, N_PER_GPU), "particles_per_timed_step": n_ref,
            "cpu_baseline": {**{k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                             "cpu_model": _cpu_model()},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def fp64_peak(device):
    import ctypes
    from paper_1411_1702_b200.sampler import load_library
    lib = load_library()
    lib.pfsmc_gpu_fp64_peak.restype = ctypes.c_int
    v = ctypes.c_double()
    rc = lib.pfsmc_gpu_fp64_peak(device, ctypes.byref(v))
    return v.value if rc == 0 else None


def gather_peak(device, n_rec=1 << 25):
    import ctypes
    from paper_1411_1702_b200.sampler import load_library
    lib = load_library()
    lib.pfsmc_gpu_gather_peak.restype = ctypes.c_int
    v = ctypes.c_double()
    rc = lib.pfsmc_gpu_gather_peak(device, ctypes.c_longlong(n_rec), ctypes.byref(v))
    return v.value if rc == 0 else None


C3_WINDOWS = (50, 200, 320)
ARITH = "exact"  # --arithmetic: the device arithmetic variant (pfsmc_gpu_config.arithmetic)
SHARD_FAILURE = []  # N > 1: why the sharded path fell back to replicas (if it did)


def _cfg(prob):
    import dataclasses
    return dataclasses.replace(prob.cfg, arithmetic=ARITH)


def _timed_steps(gpu, prob, steps, warmup, stream, j0=0, t0=0.0):
    """Blocking drop-in steps with per-step events (L2 flushed between),
    observations j0 + 1 .. j0 + warmup + steps."""
    import torch
    ms, j, tp = [], j0, t0
    iters = []
    for k in range(warmup + steps):
        j += 1
        t1 = prob.times[j - 1]
        gpu.flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
        gpu.pf_step(prob.ys[j - 1], j, tp, t1, h=prob.h_for(tp, t1))
        with torch.cuda.stream(stream):
            b.record(stream)
        torch.cuda.synchronize()
        if k >= warmup:
            ms.append(a.elapsed_time(b))
            iters.append(gpu.step_diagnostics()[2])
        tp = t1
    return ms, iters


def _cpu_ref_rate(model, prob, kw, n_cpu=1 << 14, steps=2, note=None):
    """The unmodified reference pf_step (oracle/_ref, all host threads) on a
    bounded sample of a BASELINE workload: n_cpu particles, the first `steps`
    observations (the CPU is far too slow for the full runs, and
    its throughput is flat in N)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_ctypes import REF_SO, Oracle, Reference, StepConfig
        if not os.path.exists(REF_SO):
            return {"error": "oracle/_ref not built"}
        workers = len(os.sched_getaffinity(0))
        O, R = Oracle(), Reference()
        seed = prob.cfg.seed
        sc = StepConfig(model=model, h=prob.h_for(0.0, prob.times[0]), seed=seed, **kw)
        if prob.prior_kind == "uniform":
            ens = O.init_uniform(model, n_cpu, seed, **prob.prior)
        else:
            pr = prob.prior
            ens = R.init_gaussian(sc, n_cpu, pr["th_mu"], pr["th_sigma"], pr["x_mean"], pr["x_std"],
                                  pr.get("x_clamp", [0] * len(pr["x_mean"])))
        secs, tp = 0.0, 0.0
        for j in range(1, steps + 1):
            t1 = prob.times[j - 1]
            sc.h = prob.h_for(tp, t1)
            secs += R.time_steps(sc, ens, prob.ys[j - 1:j], [t1], j, tp, workers)
            tp = t1
        out = {"value": n_cpu * steps / secs, "unit": UNIT, "cores": workers, "kind": "reference",
               "sample": f"{model} N={n_cpu}, observations 1..{steps}, reference pf_step Backend::parallel({workers})"}
        if note:
            out["note"] = note
        return out
    except Exception as e:  # noqa: BLE001  (the GPU line stands on its own)
        return {"error": repr(e)[:200]}


def _cpu_ref_windows(prob, kw, n_cpu=1 << 14):
    """C3 on the CPU: the unmodified reference pf_step (all host threads) over
    the same log-spaced grid from j = 1, timed in the same windows as the GPU.
    The reference has only the Gaussian likelihood, so it stands in for the
    lognormal extension (same propagation, which dominates the cost)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_ctypes import REF_SO, Reference, StepConfig
        if not os.path.exists(REF_SO):
            return {"error": "oracle/_ref not built"}
        workers = len(os.sched_getaffinity(0))
        R = Reference()
        seed = prob.cfg.seed
        sc = StepConfig(model="robertson", h=prob.h_for(0.0, prob.times[0]), seed=seed, **kw)
        pr = prob.prior
        ens = R.init_gaussian(sc, n_cpu, pr["th_mu"], pr["th_sigma"], pr["x_mean"], pr["x_std"], [0, 0, 0])
        timed = {j for w in C3_WINDOWS for j in range(w, w + 5)}
        secs, done, tp = 0.0, 0, 0.0
        for j in range(1, max(timed) + 1):
            t1 = prob.times[j - 1]
            sc.h = prob.h_for(tp, t1)
            dt = R.time_steps(sc, ens, prob.ys[j - 1:j], [t1], j, tp, workers)
            if j in timed:
                secs += dt
                done += 1
            tp = t1
        return {"value": n_cpu * done / secs, "unit": UNIT, "cores": workers, "kind": "reference",
                "sample": f"robertson N={n_cpu}, Gaussian likelihood, run from j=1, timed at observations "
                          + ", ".join(f"{w}..{w + 4}" for w in C3_WINDOWS)
                          + f", reference pf_step Backend::parallel({workers})"}
    except Exception as e:  # noqa: BLE001  (the GPU line stands on its own)
        return {"error": repr(e)[:200]}


def bench_workloads(local, fp64):
    """BASELINE configs 3-5 on one GPU (extra lines of the report; the
    headline metric is config 2)."""
    import numpy as np
    import torch
    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    peaks, _ = _peaks()
    hbm = float(peaks["hbm_gbs"])
    out = {}
    # config 5: resample / reduction bandwidth, 2^25 x 64-byte records
    n5 = 1 << 25
    s = GpuSampler("payload64", PfConfig(particles=n5, seed=5), ObservationModel([0], 1.0), device=local)
    rng = np.random.default_rng(0)
    s.set_ensemble(Ensemble(rng.standard_normal((n5, 6)), rng.standard_normal((n5, 2)), np.zeros(n5),
                            np.zeros(2), np.eye(2)))
    stream = torch.cuda.ExternalStream(s.stream_handle, device=local)
    by_search = {}
    for search in ("guide", "split", "bucketed"):
        s.c5_set_search(search)
        c5 = by_search[search] = {}
        for sigma in (0.1, 1.0, 4.0):
            s.c5_set_logweights(sigma, 1)
            ms = []
            for it in range(7):
                s.flush_l2()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    a.record(stream)
                s.c5_iteration(it + 1)
                with torch.cuda.stream(stream):
                    b.record(stream)
                s.synchronize()
                if it >= 2:
                    ms.append(a.elapsed_time(b))
            t = sum(ms) / len(ms)
            gbs = 184.0 * n5 / (t / 1e3) / 1e9
            c5[f"sigma={sigma}"] = {"ms_per_iteration": t, "particle_iterations_per_s": n5 / (t / 1e3),
                                   "hbm_gbs_algorithmic": gbs, "frac_of_measured_hbm": gbs / hbm}
    best = min(by_search, key=lambda k: sum(v["ms_per_iteration"] for v in by_search[k].values()))
    c5 = by_search[best]
    s.close()
    # Composite roofline for the iteration. Streamed bytes per particle (at the
    # measured HBM peak): stats 72 (the 64-byte record line + lw), exact scan
    # 33 (lg twice, cdf, segment ends), serve 68 (record write + ancestor).
    # Random bytes: two 64-byte bursts (the CDF segment and the ancestor's
    # record) at the measured random-read rate, derived from the gather
    # microbenchmark (64 B random read + 64 B streamed write per record).
    gpk = gather_peak(local)
    seq_b, rnd_b = 72 + 33 + 68, 128
    rnd_rate = 64.0 / (128.0 / (gpk * 1e9) - 64.0 / (hbm * 1e9)) if gpk else None
    bound_ms = (n5 * (seq_b / (hbm * 1e9) + rnd_b / rnd_rate) * 1e3) if rnd_rate else None
    for v in c5.values():
        v["composite_bound_ms"] = bound_ms
        v["frac_of_composite_bound"] = (bound_ms / v["ms_per_iteration"]) if bound_ms else None
    out["c5_resample_bandwidth"] = {"particles": n5, "record_bytes": 64, "bytes_per_particle_iteration": 184,
                                    "streamed_bytes_per_particle": seq_b, "random_bytes_per_particle": rnd_b,
                                    "random_gather_peak_gbs": gpk,
                                    "random_read_rate_gbs": rnd_rate / 1e9 if rnd_rate else None,
                                    "search": best, "results": c5,
                                    "results_by_search": by_search,
                                    "moments_note": "SPLIT: an iteration's gather also accumulates the weighted 2x2 moment "
                                                    "sums of the ensemble it produces (same tiles, thread layout and trees as "
                                                    "the stats pass: same bits), so from the second iteration on with unchanged "
                                                    "log-weights (the timed ones) the stats pass reads lw only; GUIDE and "
                                                    "BUCKETED read theta in the stats pass every iteration"}
    # config 3: Robertson, 2^22, BDF2 m=2, Newton <= 4, lognormal: the filter runs the
    # log-spaced grid from j = 1 and is timed in windows spread along it (early,
    # mid, stiff), since the cost per step grows with the Newton iterations
    import dataclasses
    n3 = 1 << 22
    prob = problems.robertson(particles=n3, T=400, seed=1)

    def c3_run(arith):
        g = GpuSampler("robertson", dataclasses.replace(prob.cfg, arithmetic=arith), prob.obs, device=local)
        prob.init(g)
        r = {"particles": n3, "integrator": "bdf2, m=2, newton_max_iter=4", "arithmetic": arith,
             "likelihood": "lognormal (BASELINE extension)", "windows": {}}
        st3 = torch.cuda.ExternalStream(g.stream_handle, device=local)
        j3, tp3 = 0, 0.0
        tot_ms, tot_steps, tot_it = 0.0, 0, 0.0
        for w0 in C3_WINDOWS:
            while j3 < w0 - 1:  # advance untimed to the window
                j3 += 1
                t1 = prob.times[j3 - 1]
                g.pf_step(prob.ys[j3 - 1], j3, tp3, t1, h=prob.h_for(tp3, t1))
                tp3 = t1
            ms, it = _timed_steps(g, prob, 5, 0, st3, j0=j3, t0=tp3)
            j3 += 5
            tp3 = prob.times[j3 - 1]
            t = sum(ms) / len(ms)
            ipp = float(np.mean(it)) / n3
            r["windows"][f"j={w0}..{w0 + 4}"] = {
                "t_obs": [float(prob.times[w0 - 1]), float(prob.times[w0 + 3])], "ms_per_step": t,
                "particle_steps_per_s": n3 / (t / 1e3), "newton_iterations_per_particle_step": ipp,
                "newton_iterations_per_solve": ipp / 4.0}
            tot_ms += sum(ms)
            tot_steps += len(ms)
            tot_it += float(np.sum(it))
        g.close()
        r["ms_per_step"] = tot_ms / tot_steps
        r["particle_steps_per_s"] = n3 / (r["ms_per_step"] / 1e3)
        r["newton_iterations_per_particle_step"] = tot_it / tot_steps / n3
        return r

    out["c3_robertson"] = c3 = c3_run("exact")
    c3["fast_arithmetic"] = c3_run("fast")
    c3["cpu_reference"] = _cpu_ref_windows(
        prob, dict(family="bdf", order=2, a=0.99, obs_idx=(0, 2), sigma=0.02, newton_max_iter=4))
    # config 4: 8-compartment chain, 2^24, BDF3 m=3, both arithmetic variants
    # (exact: the reference's operation order, bitwise Psi; fast: FMA and
    # reciprocals, parity at the north_star tolerances)
    import dataclasses
    n4 = 1 << 24
    prob = problems.chain8(particles=n4, T=10, seed=1)
    c4 = {}
    for arith in ("exact", "fast"):
        g = GpuSampler("chain", dataclasses.replace(prob.cfg, arithmetic=arith), prob.obs, device=local)
        prob.init(g)
        ms, it = _timed_steps(g, prob, 2, 1, torch.cuda.ExternalStream(g.stream_handle, device=local))
        g.close()
        t = sum(ms) / len(ms)
        # Newton iterations per particle-step, BOTH propagations (k_predict and
        # k_update add to one per-step counter, lmm.cpp:488 convention)
        newton = float(np.mean(it)) / n4
        # N_it(8) = 643 FP64 flops per Newton iteration (dense-LU
        # count, the reference algorithm's); the device's banded solve executes
        # fewer (EXEC_FLOPS_PER_NEWTON_CHAIN), so both are reported
        flops = 643 * newton
        tfl = flops * n4 / (t / 1e3) / 1e12
        tfl_exec = EXEC_FLOPS_PER_NEWTON_CHAIN * newton * n4 / (t / 1e3) / 1e12
        c4[arith] = {"particles": n4, "integrator": "bdf3, m=3", "arithmetic": arith, "steps": len(ms),
                     "ms_per_step": t, "particle_steps_per_s": n4 / (t / 1e3),
                     "newton_iterations_per_particle_step": newton,
                     "fp64_tflops_newton_algorithmic": tfl, "fp64_tflops_newton_executed": tfl_exec,
                     "fp64_peak_tflops_measured": fp64,
                     "frac_of_fp64_peak": (tfl / fp64) if fp64 else None,
                     "frac_of_fp64_peak_executed": (tfl_exec / fp64) if fp64 else None}
    out["c4_chain8"] = {**c4["exact"], "fast_arithmetic": c4["fast"]}
    out["c4_chain8"]["cpu_reference"] = _cpu_ref_rate(
        "chain", prob, dict(family="bdf", order=3, a=0.98, obs_idx=(0, 3, 7), sigma=0.01))
    # the reference's own problem 1 (models::MetabolicModel), BDF2 with m = 4 sub-steps,
    # N = 2^20, beside the unmodified reference pf_step on a bounded sample
    nm = 1 << 20
    prob = problems.metabolic(particles=nm, n_obs=50, seed=1)
    g = GpuSampler("metabolic", _cfg(prob), prob.obs, device=local)
    prob.init(g)
    ms, it = _timed_steps(g, prob, 5, 3, torch.cuda.ExternalStream(g.stream_handle, device=local))
    g.close()
    t = sum(ms) / len(ms)
    met = {"particles": nm, "integrator": "bdf2, h = 0.05, m = 4 per observation", "steps": len(ms),
           "ms_per_step": t, "particle_steps_per_s": nm / (t / 1e3),
           "newton_iterations_per_particle_step": float(np.mean(it)) / nm}
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_ctypes import REF_SO, Oracle, Reference, StepConfig
        if os.path.exists(REF_SO):
            workers = len(os.sched_getaffinity(0))
            O, R = Oracle(), Reference()
            n_cpu = 1 << 16
            sc = StepConfig(model="metabolic", family="bdf", order=2, h=0.05, a=0.98, seed=1, obs_idx=(0, 1, 2),
                            sigma=prob.obs.sigma)
            ens = R.init_gaussian(sc, n_cpu, prob.prior["th_mu"], prob.prior["th_sigma"], prob.prior["x_mean"],
                                  prob.prior["x_std"], prob.prior["x_clamp"])
            secs, done, tp = 0.0, 0, 0.0
            while done < 4 and secs < 10.0:
                j = done + 1
                secs += R.time_steps(sc, ens, prob.ys[j - 1:j], [prob.times[j - 1]], j, tp, workers)
                tp = prob.times[j - 1]
                done += 1
            met["cpu_reference"] = {"value": n_cpu * done / secs, "unit": UNIT, "cores": workers,
                                    "kind": "reference",
                                    "sample": f"metabolic N={n_cpu}, observations 1..{done}, reference pf_step "
                                              f"Backend::parallel({workers})"}
    except Exception as e:  # the GPU line stands on its own
        met["cpu_reference"] = {"error": repr(e)[:200]}
    out["reference_problem1_metabolic"] = met
    out["reference_problem2_advdiff"] = bench_advdiff(local, fp64)
    return out


def bench_advdiff(local, fp64, cpu=True):
    """The reference's own problem 2 (AdvDiffModel, bench.cpp:249-277 defaults:
    grid n = 20 so d = 361, 5000 particles, BDF2 at h = 0.05 i.e. m = 20 LMM
    steps per observation) and the same at 2^16 particles, with the
    unmodified reference pf_step on a bounded sample beside it."""
    import numpy as np
    import torch
    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sampler import GpuSampler
    res = {}
    for n_part, steps in ((5000, 5), (1 << 16, 3)):
        prob = problems.advdiff(particles=n_part, n=20, seed=1)
        g = GpuSampler("advdiff", prob.cfg, prob.obs, device=local, model_consts=prob.model_consts)
        prob.init(g)
        ms, it = _timed_steps(g, prob, steps, 2, torch.cuda.ExternalStream(g.stream_handle, device=local))
        g.close()
        t = sum(ms) / len(ms)
        newton = float(np.mean(it)) / n_part
        # FP64 flops per Newton iteration (advdiff.cuh): 7-point rhs (13 flops / point) + residual (4) +
        # update and norms (3) per grid point, and the DFT solve: F1 and I1 4 m H, F2 and I2 8 m H flops per
        # row / column sum term -> 24 m^2 H + the spectral multiply 6 m H
        m, H, d = 19, 10, 361
        fl_it = 20 * d + 24 * m * m * H + 6 * m * H
        tfl = fl_it * newton * n_part / (t / 1e3) / 1e12
        res[f"N={n_part}"] = {"ms_per_step": t, "particle_steps_per_s": n_part / (t / 1e3),
                              "newton_iterations_per_particle_step": newton,
                              "fp64_tflops_newton": tfl, "frac_of_fp64_peak": (tfl / fp64) if fp64 else None}
    out = {"grid_n": 20, "d": 361, "integrator": "bdf2, h = 0.05, m = 20 per observation",
           "solve": "2-D DFT diagonalisation of I - h b0 L (reference: sparse LU)", "results": res}
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_ctypes import REF_SO, Reference, StepConfig, set_advdiff_grid
        if cpu and os.path.exists(REF_SO):
            workers = len(os.sched_getaffinity(0))
            R = Reference()
            set_advdiff_grid(20, R)
            prob = problems.advdiff(particles=5000, n=20, seed=1)
            n_cpu = 4 * workers
            sc = StepConfig(model="advdiff", family="bdf", order=2, h=0.05, a=0.98, seed=1,
                            obs_idx=tuple(prob.obs.indices), sigma=prob.obs.sigma)
            ens = R.init_gaussian(sc, n_cpu, prob.prior["th_mu"], prob.prior["th_sigma"], prob.prior["x_mean"],
                                  prob.prior["x_std"], prob.prior["x_clamp"])
            secs = R.time_steps(sc, ens, prob.ys[0:1], [prob.times[0]], 1, 0.0, workers)
            R.set_model_consts()
            out["cpu_reference"] = {"value": n_cpu / secs, "unit": UNIT, "cores": workers, "kind": "reference",
                                    "sample": f"advdiff n=20 N={n_cpu}, observation 1, reference pf_step "
                                              f"Backend::parallel({workers}); Eigen's SparseLU replaced by the "
                                              "dense direct LU of oracle/ref/eigen_stub (Eigen is absent here), "
                                              "so the CPU factorisation cost is not Eigen's"}
    except Exception as e:
        out["cpu_reference"] = {"error": repr(e)[:200]}
    return out


def run_sharded(args, world, rank, local):
    """N > 1: ONE global filter of n * world particles sharded over the GPUs
    (weak scaling), NCCL collectives + ancestor migration.
    Per-step CUDA events on each rank's stream; value uses the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sharded import GpuShard, ShardedFilter, TorchComm

    if os.environ.get("PFSMC_BENCH_FORCE_SHARD_FAIL"):  # exercises the replicas fallback
        raise RuntimeError("forced sharded-path failure (PFSMC_BENCH_FORCE_SHARD_FAIL)")
    cfgno = args.config
    if cfgno == 5:
        return run_sharded_c5(args, world, rank, local)
    if cfgno == 2:    # LV, N = 2^20 per GPU (weak scaling)
        n_local = args.particles
        prob = problems.lotka_volterra(particles=n_local * world, T=T_OBS, seed=1)
        model, scaling, j_start = "lv", "weak", 0
    elif cfgno == 3:  # Robertson, N = 2^22 in total (strong), timed in the stiff part of the grid
        n_local = (1 << 22) // world
        prob = problems.robertson(particles=n_local * world, T=400, seed=1)
        model, scaling, j_start = "robertson", "strong", C3_WINDOWS[1] - 1 - args.warmup
    elif cfgno == 4:  # chain, N = 2^24 in total (strong)
        n_local = (1 << 24) // world
        prob = problems.chain8(particles=n_local * world, T=args.warmup + args.steps + 1, seed=1)
        model, scaling, j_start = "chain", "strong", 0
    else:
        raise SystemExit("--config must be 2, 3, 4 or 5")
    shard = GpuShard(model, _cfg(prob), prob.obs, rank, world, device=local)
    f = ShardedFilter([shard], TorchComm(), mode=args.shard_mode)
    prob.init(f)
    migration = "python-orchestrated, NCCL send/recv"
    if not args.python_sharded:
        shard.attach_nccl()   # the native step: one C-ABI call per observation
        migration = "native step, NCCL send/recv"
        if not args.nccl_exchange:
            try:
                if shard.attach_peers():
                    migration = "native step, pull over NVLink peer memory"
            except Exception:
                pass
    j, tp = 0, 0.0
    while j < j_start:  # untimed advance along the observation grid
        j += 1
        f.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1], prob.h_for(tp, prob.times[j - 1]))
        tp = prob.times[j - 1]
    stream = shard.stream()
    for _ in range(args.warmup):
        j += 1
        f.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1], prob.h_for(tp, prob.times[j - 1]))
        tp = prob.times[j - 1]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            shard.flush_l2()
            j += 1
            with torch.cuda.stream(stream):
                ev[k][0].record(stream)
            row = f.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1], prob.h_for(tp, prob.times[j - 1]))
            with torch.cuda.stream(stream):
                ev[k][1].record(stream)
            tp = prob.times[j - 1]
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = n_local * world * args.steps / (total_ms / 1e3)
    peaks, peak_kind = _peaks()
    hbm = float(peaks["hbm_gbs"])
    d_, p_ = shard.d, shard.p
    step_bytes = 24 * (d_ + p_ + 1) + 56  # B = 24F + 56
    step_gbs = step_bytes * n_local / (total_ms / args.steps / 1e3) / 1e9
    names = {2: "BASELINE config 2: Lotka-Volterra PF-SMC", 3: "BASELINE config 3: Robertson PF-SMC (lognormal)",
             4: "BASELINE config 4: 8-compartment chain PF-SMC"}
    mode_txt = ("exact-mode ancestor migration (bitwise the single filter; (G-1)/G of the slots fetch a remote "
                "ancestor)" if args.shard_mode == "exact" else
                "offspring-allocation migration (per-particle offspring counts bitwise the single filter's; "
                "children built on the ancestor's GPU; only the load imbalance crosses GPUs)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded {prob.name} observations)",
            "config": {"workload": names[cfgno], "particles_per_gpu": n_local,
                       "global_particles": n_local * world, "first_timed_observation": j - args.steps + 1,
                       "shrink_a": prob.cfg.shrink_a, "arithmetic": ARITH,
                       "integrator": f"{prob.cfg.family}{prob.cfg.order} (m={prob.substeps})",
                       "l2": "flushed between timed steps", "shard_mode": args.shard_mode,
                       "parallelism": f"sharded x{world}: one global filter, NCCL allgathers + {mode_txt} "
                                      f"({migration})"},
            "roofline": {"bound": "hbm", "kernel": "whole step", "achieved": step_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": step_gbs / hbm, "traffic": None, "bytes_per_particle": step_bytes,
                         "peak_source": peak_kind},
            "gpu_launches": 12 * args.steps,
            "e2e": {"value": n_local * world * args.steps / t_wall, "unit": UNIT,
                    "h2d_bytes_per_step": shard.transfer_bytes()[0], "d2h_bytes_per_step": shard.transfer_bytes()[1],
                    "path": "ShardedFilter.pf_step (host y in, trace out)"},
            "clocks": clk.summary(),
            "final_trace": {"theta_mean": list(map(float, row.theta_mean)), "ess": float(row.ess)}}
    if rank == 0:
        print(json.dumps(line))
    shard.close()
    dist.destroy_process_group()
    return 0


def run_sharded_c5(args, world, rank, local):
    """BASELINE config 5 over N GPUs: 2^25 64-byte records per GPU (weak
    scaling, 2^28 at N = 8), one global resample / reduction iteration per
    step: LSE + weighted 2x2 covariance (group partials allgathered), the
    exact scan over all shards, the exact multinomial and the gather with the
    records of other GPUs pulled over NVLink peer memory (exact migration).
    Device time per iteration (CUDA events, max over ranks); NVLink bytes from
    the device count of records pulled from other GPUs."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1411_1702_b200.sampler import Ensemble, ObservationModel, PfConfig
    from paper_1411_1702_b200.sharded import GpuShard, ShardedFilter, TorchComm

    n_local = 1 << 25 if args.particles == N_PER_GPU else args.particles
    shard = GpuShard("payload64", PfConfig(particles=n_local * world, seed=5), ObservationModel([0], 1.0), rank, world,
                     device=local)
    f = ShardedFilter([shard], TorchComm(), pull=True)
    rng = np.random.default_rng(1000 + rank)
    shard.set_ensemble(Ensemble(rng.standard_normal((n_local, 6)), rng.standard_normal((n_local, 2)),
                                np.zeros(n_local), np.zeros(2), np.eye(2)))
    f._refresh(0)  # the global shrink mean of the injected records
    shard.attach_nccl()
    peers = shard.attach_peers()
    if not peers:
        raise SystemExit("config 5 sharded: the peer-memory mapping failed")
    stream = shard.stream()
    res = {}
    total_all, remote_all, its_all = 0.0, 0, 0
    with ClockSampler(local) as clk:
        for sigma in (0.1, 1.0, 4.0):
            shard.c5_set_logweights(sigma, 1)
            for it in range(args.warmup):
                f.c5_iteration(it + 1)
            shard.synchronize()
            r0 = shard.c5_remote_pulls()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            dist.barrier()
            torch.cuda.synchronize()
            for k in range(args.steps):
                shard.flush_l2()
                with torch.cuda.stream(stream):
                    ev[k][0].record(stream)
                f.c5_iteration(args.warmup + k + 1)
                with torch.cuda.stream(stream):
                    ev[k][1].record(stream)
            shard.synchronize()
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev)
            t = torch.tensor([ms], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            remote = shard.c5_remote_pulls() - r0
            rt = torch.tensor([remote], dtype=torch.int64, device=f"cuda:{local}")
            dist.all_reduce(rt)
            remote = int(rt.item())
            per_it = ms / args.steps
            res[f"sigma={sigma}"] = {
                "ms_per_iteration": per_it,
                "particle_iterations_per_s": n_local * world / (per_it / 1e3),
                "hbm_gbs_per_gpu_algorithmic": 184.0 * n_local / (per_it / 1e3) / 1e9,
                "remote_records_per_iteration": remote / args.steps,
                "nvlink_record_gbs_per_gpu": 64.0 * remote / args.steps / world / (per_it / 1e3) / 1e9}
            total_all += ms
            remote_all += remote
            its_all += args.steps
    per_it = total_all / its_all
    peaks, peak_kind = _peaks()
    hbm = float(peaks["hbm_gbs"])
    value = n_local * world / (per_it / 1e3)
    gbs = 184.0 * n_local / (per_it / 1e3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "particle-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_it, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (N(0,1) records, lw ~ N(0, sigma^2))",
            "config": {"workload": "BASELINE config 5: resample/reduction bandwidth microbenchmark",
                       "particles_per_gpu": n_local, "global_particles": n_local * world, "record_bytes": 64,
                       "sigmas": [0.1, 1.0, 4.0], "l2": "flushed between timed iterations",
                       "parallelism": f"sharded x{world}: group-partial allgathers, exact scan over all shards, "
                                      "exact-mode migration pulled over NVLink peer memory"},
            "roofline": {"bound": "hbm", "kernel": "whole iteration", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                         "frac": gbs / hbm, "traffic": None, "bytes_per_particle": 184, "peak_source": peak_kind},
            "nvlink_record_gbs_per_gpu": 64.0 * remote_all / its_all / world / (per_it / 1e3) / 1e9,
            "results": res, "gpu_launches": 8 * its_all, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line))
    shard.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--particles", type=int, default=N_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of sharding")
    ap.add_argument("--python-sharded", action="store_true",
                    help="sharded path orchestrated phase by phase from Python (default: native NCCL step)")
    ap.add_argument("--nccl-exchange", action="store_true",
                    help="migrate with counted NCCL send/recv instead of the peer-memory pull")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the sharded path (NCCL collectives + migration) even at N = 1 (a check of that path)")
    ap.add_argument("--no-workloads", action="store_true", help="skip the configs 3-5 extra lines")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE config for N > 1 (sharded) runs; the single-GPU line is config 2 with 3-5 as "
                         "workload extras")
    ap.add_argument("--shard-mode", default="offspring", choices=["exact", "offspring"],
                    help="sharded migration mode (pfsmc_gpu_shard_set_mode)")
    ap.add_argument("--arithmetic", default="exact", choices=["exact", "fast"],
                    help="device arithmetic: exact (reference op order, bitwise Psi) or fast (FMA; tolerance parity)")
    args = ap.parse_args()
    global ARITH
    ARITH = args.arithmetic
    world, rank, local = _dist()
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import numpy as np
    import torch

    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sampler import GpuSampler

    if args.warmup < 3:
        args.warmup = 3
    torch.cuda.set_device(local)
    if world > 1 or args.force_sharded:
        import torch.distributed as dist
        if "MASTER_ADDR" not in os.environ:  # a plain single-process run with --force-sharded
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]), RANK="0",
                              WORLD_SIZE="1")
            sk.close()
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        if not args.replicas:
            try:
                return run_sharded(args, world, rank, local)
            except Exception as e:  # noqa: BLE001
                # the scaling line must still be produced: independent replicas
                # (no collectives in the data path), with the failure recorded
                print(f"[bench] sharded path failed on rank {rank}: {e!r}; falling back to replicas",
                      file=sys.stderr, flush=True)
                SHARD_FAILURE.append(repr(e)[:300])
                if not dist.is_initialized():
                    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    n = args.particles
    T = min(T_OBS, 2 * args.steps + args.warmup + args.e2e_steps + 4)
    prob = problems.lotka_volterra(particles=n, T=T_OBS, seed=1)
    # replicas: every rank filters its own N-particle ensemble
    cfg = _cfg(prob)
    gpu = GpuSampler("lv", cfg, prob.obs, device=local)
    gpu.initialize_uniform(**prob.prior)
    gpu.upload_observations(prob.ys[:T], prob.times[:T], 0.0)
    stream = torch.cuda.ExternalStream(gpu.stream_handle, device=local)

    j = 0
    for _ in range(args.warmup):
        j += 1
        gpu.step_resident(j)
    gpu.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # headline: the production path (one CUDA graph per step, programmatic
    # dependent launches between the five kernels), events around each step
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            gpu.flush_l2()
            j += 1
            with torch.cuda.stream(stream):
                ev[k][0].record(stream)
            gpu.step_resident(j)
            with torch.cuda.stream(stream):
                ev[k][1].record(stream)
        last = gpu.synchronize()
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # per-kernel breakdown (and the roofline's kernel duration): a second pass
    # of the same steps with events between the kernels (no graph, no PDL)
    gpu.set_kernel_timing(True)
    for k in range(args.steps):
        gpu.flush_l2()
        j += 1
        gpu.step_resident(j)
    gpu.synchronize()
    kt = gpu.kernel_times()
    gpu.set_kernel_timing(False)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = n * world * args.steps / (total_ms / 1e3)

    # e2e: the drop-in C-ABI pf_step with host buffers (y in, trace row out)
    ys_pinned = torch.tensor(prob.ys[:T], dtype=torch.float64).pin_memory().numpy()
    e2e_s = 0.0
    e2e_steps = max(1, min(args.e2e_steps, T - j))
    for _ in range(e2e_steps):
        j += 1
        gpu.flush_l2()
        gpu.synchronize()
        t0 = time.perf_counter()
        gpu.pf_step(ys_pinned[j - 1], j, prob.times[j - 2], prob.times[j - 1])
        e2e_s += time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d, d2h = gpu.transfer_bytes()
    e2e = {"value": n * world * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": e2e_steps,
           "bytes_note": "StepParams up (y, times, constants), DevState down (trace row, error word, moments)",
           "path": "pfsmc_gpu_step (C ABI drop-in for filter::pf_step), blocking"}

    # the literal drop-in, pfsmc_gpu::pf_step(Ensemble&, ...) (include/pfsmc_gpu.hpp):
    # the whole host ensemble in and out every step, as filter::pf_step mutates
    # the caller's Ensemble (filter.cpp:332, 373-377)
    lit_s, lit_steps = 0.0, 3
    host_ens = gpu.get_ensemble()
    for _ in range(lit_steps):
        j += 1
        gpu.synchronize()
        t0 = time.perf_counter()
        gpu.set_ensemble(host_ens)
        gpu.pf_step(ys_pinned[j - 1], j, prob.times[j - 2], prob.times[j - 1])
        gpu.get_ensemble(out=host_ens)  # in place, as filter::pf_step mutates the caller's Ensemble
        lit_s += time.perf_counter() - t0
    ens_bytes = 8 * n * (D + P + 1) + 8 * (P + P * P)
    e2e["literal_ensemble_step"] = {
        "value": n * lit_steps / lit_s, "unit": UNIT, "steps": lit_steps,
        "h2d_bytes_per_step": ens_bytes + h2d, "d2h_bytes_per_step": ens_bytes + d2h,
        "path": "set_ensemble + pfsmc_gpu_step + get_ensemble: the Ensemble& drop-in (pfsmc_gpu.hpp pf_step), "
                "host AoS ensemble copied and transposed both ways every step"}
    peaks, peak_kind = _peaks()
    hbm = float(peaks["hbm_gbs"])
    names = list(kt.keys())
    dom = max(names, key=lambda k: kt[k])
    avg_ms = kt[dom] / args.steps
    achieved = KERNEL_BYTES[dom] * n / (avg_ms / 1e3) / 1e9
    traffic, prof = None, {}
    tpath = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    if os.path.exists(tpath):
        try:
            prof = json.load(open(tpath)).get(dom, {})
            traffic = prof.get("dram_bytes_per_launch")
        except Exception:
            traffic, prof = None, {}
    step_gbs = STEP_BYTES * n / (total_ms / args.steps / 1e3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded RK4 Lotka-Volterra observations, uniform priors)",
            "config": {**_lv_config(world, n),
                       **({"sharded_path_failed": SHARD_FAILURE[0]} if SHARD_FAILURE else {})},
            "arithmetic": ARITH,
            "exact_scan": "single pass (k_scan_fused: decoupled look-back); the two-pass form serves the sharded step",
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "bytes_per_particle": KERNEL_BYTES[dom], "peak_source": peak_kind,
                         # what actually limits the kernel (one ncu --set full capture of this
                         # command, profiles/kernel_traffic.json): instruction issue, not HBM
                         "ncu_issue_active_pct": prof.get("issue_active_pct"),
                         "ncu_fp64_pipe_pct": prof.get("fp64_pipe_pct"),
                         "ncu_achieved_occupancy_pct": prof.get("achieved_occupancy_pct"),
                         "ncu_source": prof.get("source"),
                         # the instruction-issue floor of the same kernel: its warp instructions
                         # (ncu) at one issue per scheduler per cycle, 4 schedulers x the SMs, at
                         # the sampled SM clock; frac_of_issue_floor = floor / measured duration
                         **_issue_floor(prof, avg_ms, clk.summary())},
            "step_roofline": {"bytes_per_particle": STEP_BYTES, "achieved": step_gbs, "peak": hbm,
                              "frac": step_gbs / hbm},
            "kernel_ms_per_step": {k: v / args.steps for k, v in kt.items()},
            "gpu_launches": len(kt) * args.steps,
            "e2e": e2e, "clocks": clk.summary(),
            "final_trace": {"theta_mean": list(map(float, last[:P])), "ess": float(last[-1])}}
    # the same resident graph step with the FAST arithmetic variant (FMA,
    # reciprocals; parity at the north_star tolerances, tests/test_gpu_parity.py
    # fast_* cases) on its own handle, same seed / observations
    if world == 1 and ARITH == "exact":
        import dataclasses
        gf = GpuSampler("lv", dataclasses.replace(cfg, arithmetic="fast"), prob.obs, device=local)
        gf.initialize_uniform(**prob.prior)
        gf.upload_observations(prob.ys[:T], prob.times[:T], 0.0)
        sf = torch.cuda.ExternalStream(gf.stream_handle, device=local)
        jf = 0
        for _ in range(args.warmup):
            jf += 1
            gf.step_resident(jf)
        gf.synchronize()
        evf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            gf.flush_l2()
            jf += 1
            with torch.cuda.stream(sf):
                evf[k][0].record(sf)
            gf.step_resident(jf)
            with torch.cuda.stream(sf):
                evf[k][1].record(sf)
        gf.synchronize()
        torch.cuda.synchronize()
        fms = sum(a.elapsed_time(b) for a, b in evf) / args.steps
        gf.close()
        line["fast_arithmetic"] = {"value": n / (fms / 1e3), "unit": UNIT, "ms_per_step": fms,
                                   "note": "same workload, PFSMC_GPU_ARITH_FAST handle (FMA contraction, reciprocal "
                                           "multiplies); the headline value is the exact (reference operation "
                                           "order) build"}
    fp64 = fp64_peak(local)
    line["fp64_peak_tflops_measured"] = fp64
    if world == 1 and not args.no_workloads:
        try:
            line["workloads"] = bench_workloads(local, fp64)
        except Exception as e:  # the headline line must still print
            line["workloads"] = {"error": repr(e)[:300]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(N_PER_GPU, 20, 15.0, len(os.sched_getaffinity(0)), prob)
        line["cpu_baseline"] = {**{k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                                "cpu_model": _cpu_model(), "sequential": cpu_sequential(prob)}
    if rank == 0:
        print(json.dumps(line))
    gpu.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
