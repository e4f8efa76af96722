"""Fused (single-pass, look-back) vs two-pass exact scan: the LV 2^20 headline
step (resident graph step, events, L2 flushed between) and the config-5
iteration at 2^25, same process, alternating.
    python profiles/probe_scanmode.py [lv] [c5]"""
import dataclasses
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1411_1702_b200 import problems  # noqa: E402
from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig  # noqa: E402


def timed(g, fn, reps):
    st = torch.cuda.ExternalStream(g.stream_handle)
    ms = []
    for r in range(reps):
        g.flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
        fn(r)
        with torch.cuda.stream(st):
            b.record(st)
        g.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms), min(ms)


def lv(out):
    n = 1 << 20
    prob = problems.lotka_volterra(particles=n, T=400, seed=1)
    g = GpuSampler("lv", prob.cfg, prob.obs)
    g.initialize_uniform(**prob.prior)
    g.upload_observations(prob.ys[:400], prob.times[:400], 0.0)
    j = [1]

    def step(_):
        g.step_resident(j[0])
        j[0] += 1

    for _ in range(5):
        step(0)
    g.synchronize()
    res = {}
    for rnd in range(3):
        for mode in ("fused", "two_pass"):
            g.set_scan_mode(mode)
            step(0)
            g.synchronize()
            res.setdefault(mode, []).append(timed(g, step, 30)[0])
    for mode in ("fused", "two_pass"):
        g.set_scan_mode(mode)
        g.set_kernel_timing(True)
        k0 = g.kernel_times()
        for _ in range(10):
            step(0)
        g.synchronize()
        k1 = g.kernel_times()
        g.set_kernel_timing(False)
        out[f"lv_{mode}"] = {"ms_per_step": statistics.median(res[mode]), "rounds": res[mode],
                             "kernel_us": {k: (k1[k] - k0.get(k, 0.0)) / 10 * 1000 for k in k1}}
        # (kernel-time counters accumulate across modes: names change with the mode, so subtract by name)
    g.close()


def c5(out):
    n = 1 << 25
    s = GpuSampler("payload64", PfConfig(particles=n, seed=77), ObservationModel([0], 1.0))
    from paper_1411_1702_b200.sampler import Ensemble
    rng = np.random.default_rng(0)
    s.set_ensemble(Ensemble(rng.standard_normal((n, 6)), rng.standard_normal((n, 2)), np.zeros(n),
                            np.zeros(2), np.eye(2)))
    s.c5_set_search("split")
    for sigma in (0.1, 1.0, 4.0):
        s.c5_set_logweights(sigma, 5)
        for mode in ("fused", "two_pass", "fused", "two_pass"):
            s.set_scan_mode(mode)
            s.c5_set_logweights(sigma, 5)
            s.c5_iteration(1)
            s.synchronize()

            def it(r):
                s.c5_iteration(2 + r)

            # weights are not regenerated between iterations here: the scan, search and gather costs
            # do not depend on which records sit in the slots
            med, mn = timed(s, it, 10)
            out.setdefault(f"c5_sigma{sigma}_{mode}", []).append(med)
    s.close()


if __name__ == "__main__":
    which = sys.argv[1:] or ["lv", "c5"]
    out = {}
    if "lv" in which:
        lv(out)
    if "c5" in which:
        c5(out)
    print(json.dumps(out, indent=1))
