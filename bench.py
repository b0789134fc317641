#!/usr/bin/env python
"""bench.py -- S-Merge throughput on B200 at BASELINE.json config 2.

Workload (BASELINE.json configs[1]): symmetric merge of two k=20
subgraphs of 500,000 points each; d=128 fp32 from a 1,000-component
Gaussian mixture (centres U[0,255], sigma 20) clipped to [0,255] and
rounded; L2.  Synthetic, seeded data stands in for SIFT1M.
The subgraphs are built first (untimed) with this package's NN-Descent,
which is bit-identical to the reference's.

One step = one full ``s_merge`` call (split, random cross appends, every
local-join round to convergence, export, rear merge).

  value  distance evaluations/s with the dataset and both subgraphs already
         resident in HBM and the result left in HBM (CUDA events on the
         engine stream).
  e2e    the same metric through the public API with host numpy inputs:
         dataset upload, graph upload, result download inside the region.

``--impl reference`` times the CPU oracle (oracle/, a C/OpenMP restatement
of the reference's numba kernels; the Python reference cannot travel to the
GPU box) on a bounded sample of the same workload with all host cores.
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

CFG = dict(n=1_000_000, d=128, k=20, r=0.5, n_centres=1000, sigma=20.0, data_seed=7,
           split_seed=1, g_seed=1, h_seed=2, merge_seed=3)
CPU_SAMPLE_N = 100_000  # 2 x 50k points of the same distribution

# BASELINE.json configs: data generator, metric, k, operation.
# Subgraphs / the built graph come from this package's NN-Descent (bit-exact
# to the reference's), seeds 1 and 2; merge seed 3; halves of a seeded
# permutation (split seed 1).  c5l1 is one level-1 merge of config 5's tree
# (two 1M-point subgraphs, ids [0, 1M) and [1M, 2M), subgraph seeds 1, 2).
CONFIGS = {
    "c1": dict(n=10_000, d=32, k=20, metric="l2", op="s", gen="uniform", gen_seed=1,
               split="halves", max_iters=10, min_update_fraction=0.0),
    "c2": dict(n=1_000_000, d=128, k=20, metric="l2", op="s", gen="int_gmm", centres=1000,
               sigma=20.0, gen_seed=7, split="perm"),
    "c3": dict(n=1_000_000, d=960, k=20, metric="l2", op="j", gen="unit_gmm", centres=500,
               sigma=0.05, gen_seed=7, split="perm"),
    "c4": dict(n=1_200_000, d=100, k=40, metric="cosine", op="s", gen="sphere_gmm", centres=2000,
               sigma=0.3, gen_seed=7, split="perm"),
    "c5l1": dict(n=2_000_000, d=128, k=20, metric="l2", op="s", gen="int_gmm", centres=1000,
                 sigma=20.0, gen_seed=7, split="halves"),
}


def config_inputs(km, name, scale=1.0):
    """(dataset, metric, k, op, s1, s2, merge-param kwargs) of a BASELINE config."""
    c = CONFIGS[name]
    n = max(int(c["n"] * scale), 64)
    if c["gen"] == "uniform":
        ds = km.generate_uniform(n, c["d"], seed=c["gen_seed"])
    else:
        gen = {"int_gmm": km.generate_int_gmm, "unit_gmm": km.generate_unit_gmm,
               "sphere_gmm": km.generate_sphere_gmm}[c["gen"]]
        ds = gen(n, c["d"], n_centres=c["centres"], sigma=c["sigma"], seed=c["gen_seed"])
    if c["split"] == "halves":
        s1, s2 = np.arange(n // 2, dtype=np.int64), np.arange(n // 2, n, dtype=np.int64)
    else:
        s1, s2 = split_ids(n, 1)
    metric = km.Metric.L2 if c["metric"] == "l2" else km.Metric.COSINE
    mp = {key: c[key] for key in ("max_iters", "min_update_fraction") if key in c}
    return ds, metric, c["k"], c["op"], s1, s2, mp
REF_BUDGET_S = 1500.0  # reference arm: whole-run bound (setup + timed steps)
METRIC = "distance_evals_per_s"
UNIT = "evals/s"


def split_ids(n, seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    h = n // 2
    return np.sort(perm[:h]), np.sort(perm[h:])


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (the
    profiling recipe's clocks line: clocks.sm, clocks.max.sm, hw_slowdown,
    hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap).  Sampled through
    NVML from a host thread every 100 ms: an `nvidia-smi -lms` loop stalled
    the step it landed in (by 2-12 ms, once by 200 ms), which the timed
    region would include.  Falls back to nvidia-smi when NVML is missing."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    PERIOD_S = 0.1

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._p = None
        self._nvml = None

    def _nvml_handle(self):
        import pynvml as N

        N.nvmlInit()
        try:
            import torch

            pr = torch.cuda.get_device_properties(self.device)
            bus = "%08X:%02X:%02X.0" % (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
            return N, N.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return N, N.nvmlDeviceGetHandleByIndex(self.device)

    def _nvml_sample(self):
        N, h = self._nvml
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap)
        return [str(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                str(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))] + \
            ["Active" if r & b else "Not Active" for b in bits]

    def __enter__(self):
        import threading

        self._lines = []
        self._stop = threading.Event()
        try:
            self._nvml = self._nvml_handle()
            self.samples.append(self._nvml_sample())  # before the region

            def poll():
                while not self._stop.wait(self.PERIOD_S):
                    self.samples.append(self._nvml_sample())

            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            self._nvml = None
        self._first = threading.Event()
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def reader():
                for line in self._p.stdout:
                    self._lines.append(line)
                    self._first.set()
                self._first.set()

            self._t = threading.Thread(target=reader, daemon=True)
            self._t.start()
            # nvidia-smi's start-up must not overlap the timed region
            self._first.wait(timeout=15)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._nvml is not None:
            self._stop.set()
            self._t.join(timeout=5)
            try:
                self.samples.append(self._nvml_sample())  # at the end of the region
                self._nvml[0].nvmlShutdown()
            except Exception:
                pass
            return
        if self._p is None:
            return
        time.sleep(0.25)  # one more sample from inside / at the end of the region
        self._p.terminate()
        try:
            self._p.wait(timeout=10)
        except Exception:
            self._p.kill()
        self._t.join(timeout=5)
        for line in self._lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_inputs(km, n):
    ds = km.generate_int_gmm(n, CFG["d"], n_centres=CFG["n_centres"], sigma=CFG["sigma"],
                             seed=CFG["data_seed"])
    s1, s2 = split_ids(n, CFG["split_seed"])
    return ds, s1, s2


def recall_sample(ds, graph, device, nq=1000, seed=0, metric=None):
    """recall@10 of `graph` on nq sampled nodes against exact brute force
    (the package's GPU brute force: exact fp64 distances, (dist, id) order,
    self excluded -- reference brute_force_queries semantics)."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    rng = np.random.default_rng(seed)
    q = np.sort(rng.choice(ds.n, size=min(nq, ds.n), replace=False))
    eng = get_engine(device)
    eng.set_dataset(ds.vectors, int(km.Metric.L2 if metric is None else metric))
    ids, _ = eng.bf_topk(11, queries=ds.vectors[q])
    truth = [[int(v) for v in row if v != qq][:10] for row, qq in zip(ids, q)]
    rows = np.searchsorted(np.asarray(graph.member_ids), q)
    got = np.asarray(graph.ids)[rows, :10]
    hits = sum(len(set(t) & set(g.tolist())) for t, g in zip(truth, got))
    return hits / (len(q) * 10)


def cpu_baseline(n_sample=CPU_SAMPLE_N):
    """Oracle S-Merge on a bounded sample (2 x n/2 points, same distribution)."""
    from oracle import oracle as O
    import paper_1908_00814_b200.core as core

    O.build()
    ds = core.generate_int_gmm(n_sample, CFG["d"], n_centres=CFG["n_centres"],
                               sigma=CFG["sigma"], seed=CFG["data_seed"])
    s1, s2 = split_ids(n_sample, CFG["split_seed"])
    g, _, _ = O.nn_descent(ds.vectors, 1, CFG["k"], CFG["g_seed"], member_ids=s1)
    h, _, _ = O.nn_descent(ds.vectors, 1, CFG["k"], CFG["h_seed"], member_ids=s2)
    t0 = time.perf_counter()
    u, rep, count = O.s_merge(ds.vectors, g, h, CFG["k"], r=CFG["r"], seed=CFG["merge_seed"])
    dt = time.perf_counter() - t0
    return dict(value=count / dt, seconds=dt, evals=count, rounds=len(rep.rounds),
                cores=os.cpu_count(), kind="port",
                sample=f"s_merge of 2x{n_sample // 2} points, config-2 distribution, k=20; "
                       "subgraphs built by the oracle's nn_descent (untimed)")


def run_reference(args):
    """The reference arm: the CPU oracle (oracle/, the C/OpenMP restatement of
    the reference's numba kernels, all host threads) on the SAME workload as
    the GPU arm -- the full config-2 S-Merge (2 x 500,000 points) per step.
    The subgraphs are built by the oracle's own NN-Descent (untimed).  The
    oracle has no JIT, so warm-up steps run on a 2 x 5,000 sample; if the
    projected run would exceed REF_BUDGET_S, fewer full steps are timed and
    ``steps_timed`` says how many (the driver's step limit is 1,800 s)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from oracle import oracle as O
    import paper_1908_00814_b200.core as core

    O.build()
    n = int(CFG["n"] * args.scale)
    t_setup = time.perf_counter()
    ds = core.generate_int_gmm(n, CFG["d"], n_centres=CFG["n_centres"], sigma=CFG["sigma"],
                               seed=CFG["data_seed"])
    s1, s2 = split_ids(n, CFG["split_seed"])
    g, _, _ = O.nn_descent(ds.vectors, 1, CFG["k"], CFG["g_seed"], member_ids=s1)
    h, _, _ = O.nn_descent(ds.vectors, 1, CFG["k"], CFG["h_seed"], member_ids=s2)
    setup_s = time.perf_counter() - t_setup
    wn = 10_000
    wds = core.generate_int_gmm(wn, CFG["d"], n_centres=CFG["n_centres"], sigma=CFG["sigma"],
                                seed=CFG["data_seed"])
    w1, w2 = split_ids(wn, CFG["split_seed"])
    wg, _, _ = O.nn_descent(wds.vectors, 1, CFG["k"], CFG["g_seed"], member_ids=w1)
    wh, _, _ = O.nn_descent(wds.vectors, 1, CFG["k"], CFG["h_seed"], member_ids=w2)
    for _ in range(args.warmup):
        O.s_merge(wds.vectors, wg, wh, CFG["k"], r=CFG["r"], seed=CFG["merge_seed"])
    evals, done, step_s = 0, 0, []
    t0 = time.perf_counter()
    for i in range(args.steps):
        ts = time.perf_counter()
        _, rep, count = O.s_merge(ds.vectors, g, h, CFG["k"], r=CFG["r"], seed=CFG["merge_seed"])
        step_s.append(round(time.perf_counter() - ts, 3))
        evals += count
        done += 1
        el = time.perf_counter() - t0
        if el + el / done > REF_BUDGET_S - setup_s:
            break
    dt = time.perf_counter() - t0
    v = evals / dt
    sample = (f"the full workload: s_merge of 2x{n // 2} points (config-2 distribution, k=20) "
              "per step; oracle C/OpenMP restatement of the reference kernels, subgraphs from "
              "the oracle's nn_descent")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "steps_timed": done, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / done, "merge_seconds": dt / done, "step_seconds": step_s,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "config2_smerge_2x500k_d128_k20",
                                            "n": n, "d": CFG["d"], "k": CFG["k"], "r": CFG["r"],
                                            "metric": "l2", "rho": 1.0, "sample_points": n,
                                            "parallelism": "host threads"},
            "same_config": n == CFG["n"], "setup_seconds": setup_s,
            "evals_per_step": evals // done, "rounds": len(rep.rounds),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def kernel_rooflines(st, steps, d, k, slot_b, lazy, hbm_peak, row_b=None, cosine=False):
    """Algorithmic-byte rooflines of the join, apply and assembly kernels of
    one step, from the run's own counters (SURVEY.md §8d's byte model):

    join      (row_b + 4) * sum|M_u| + slot_b * written_slots
              (exact fp64 evaluations in the join read the rows already
              staged in shared memory: no HBM bytes of their own; they are
              reported against the fp64 pipe instead, ``fp64`` below)
    apply     8 * slots read + (slot_b - 8) * written slots (source ids)
              + 13 k per row loaded + 13 k per row stored (ids, dists, flags)
              (+ 4 d per lazy exact evaluation in the apply: the candidate row)
    assemble  9 k per active hood (forward ids + flags, reverse entries)
              + 20 B per membership (hood entry + membership record)

    ``row_b``: bytes per gathered member row (default fp32 rows, 4 d)."""
    row_b = 4.0 * d if row_b is None else float(row_b)
    ex_apply = 4.0 * d * st["exact_evals"] if lazy else 0.0
    out = {}
    jb = (row_b + 4.0) * st["members"] + slot_b * st["written_slots"]
    ab = (8.0 * st["candidates"] + (slot_b - 8.0) * st["written_slots"]
          + 13.0 * k * (st["apply_rows_in"] + st["apply_rows_out"]) + ex_apply)
    for name, b, ms in (("join", jb, st["join_kernel_ms"]), ("apply", ab, st["apply_kernel_ms"])):
        gbs = b / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        out[name] = {"bytes_per_step": b / steps, "ms_per_step": ms / steps, "achieved": gbs,
                     "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak}
    if st["exact_evals"] > 0:
        # exact reference sums: d dependent fp64 steps per evaluation, 3 fp64
        # instructions per dimension (sub, mul, add; 2 for the cosine dot),
        # against 64 fp64 lanes x 148 SMs x 1.965 GHz (nominal, non-FMA)
        ops = float(st["exact_evals"]) * d * (2.0 if cosine else 3.0)
        ms = st["apply_kernel_ms"] if lazy else st["join_kernel_ms"]
        peak = 64 * 148 * 1.965e9
        out["apply" if lazy else "join"]["fp64"] = {
            "exact_evals_per_step": st["exact_evals"] / steps,
            "lazy_batches_per_step": st["lazy_batches"] / steps, "ops_per_step": ops / steps,
            "achieved_tops": ops / (ms / 1e3) / 1e12, "peak_tops": peak / 1e12,
            "frac": ops / (ms / 1e3) / peak, "peak_kind": "nominal"}
    return out


def config_legs(km, names, device, steps, warmup, hbm_peak, no_recall=False):
    """BASELINE configs beyond the headline (c3: J-Merge d=960 lazy route;
    c4: cosine k=40 S-Merge), device-resident inputs, timed with CUDA events
    on the engine stream: merge seconds, evals/s, exact evaluations and the
    join / apply rooflines (fp32 byte model, §8d)."""
    import torch

    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine(device)
    res = {}
    for name in names:
        t = time.perf_counter()
        ds, metric, k, op, s1, s2, mpk = config_inputs(km, name)
        g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1, device=device,
                          out_device=True)
        h = (km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2, device=device,
                           out_device=True) if op == "s" else None)
        setup = time.perf_counter() - t
        params = km.MergeParams(k=k, seed=3, **mpk)

        def run(c):
            if op == "s":
                return km.s_merge(ds, g, h, params, counter=c, device=device, out_device=True)
            return km.j_merge(ds, g, s2, params, counter=c, device=device, out_device=True)

        u = None
        for _ in range(max(1, warmup)):
            u = run(km.DistanceCounter())
        del u
        torch.cuda.synchronize(device)
        eng.reset_stats()
        eng.set_profiling(True)
        evals = 0
        eng.mark(6)
        for _ in range(steps):
            c = km.DistanceCounter()
            u = run(c)
            evals += c.count
        eng.mark(7)
        ms = eng.elapsed_ms(6, 7)
        st = eng.stats()
        eng.set_profiling(False)
        inf = eng.info()
        lazy = (not inf["cert"]) and ds.d > 384
        slot_b = 8.0 if (inf["cert"] or inf["cert_dot"]) else 12.0
        tc = st["tc_join_launches"] > 0
        dense = st["dense_join_launches"] > 0
        # k_join_tc gathers three u8 limb planes per row (3 bytes per dimension,
        # rows padded to 16), not the fp32 row: the byte model follows the kernel
        row_b = 3.0 * ((ds.d + 15) // 16 * 16) if tc else None
        kr = kernel_rooflines(st, steps, ds.d, k, slot_b, lazy, hbm_peak, row_b=row_b,
                              cosine=int(metric) == 2)
        kr["join"]["bytes_model"] = (
            "3-byte fixed-point limb rows (k_join_tc) + hood entries + 12 B per written slot" if tc else
            "fp32 rows (4 d, SURVEY 8d) + hood entries + slot bytes; k_join_dense actually gathers "
            "fp64 rows (8 d) and a per-hood record" if dense else
            "fp32 rows (4 d, SURVEY 8d) + hood entries + slot bytes")
        rec = None
        if not no_recall:
            uh = km.KnnGraph.from_arrays(u.member_ids, u.k, u.metric, u.ids.cpu().numpy(),
                                         u.dists.cpu().numpy(), u.sizes.cpu().numpy())
            rec = recall_sample(ds, uh, device, metric=metric)
        res[name] = {
            "workload": {"c3": "config3_jmerge_500k+500k_d960_k20",
                         "c4": "config4_smerge_2x600k_d100_k40_cosine"}.get(name, name),
            "merge_seconds": ms / steps / 1e3, "evals_per_step": evals // steps,
            "evals_per_s": evals / (ms / 1e3), "steps": steps,
            "rounds_per_step": st["rounds"] / steps,
            "exact_evals_per_step": st["exact_evals"] / steps,
            "exact_fraction": st["exact_evals"] / max(1, st["pairs"]),
            "route": ("lazy: tcgen05 fixed-point lower bounds in the join (k_join_tc), exact fp64 in the apply"
                      if lazy and tc else
                      "lazy (d-chunked fp32 join, exact fp64 in the apply)" if lazy else
                      "tensor-core (mma.sync, certified)" if inf["cert_dot"] else
                      "dense exact fp64 register tiles (k_join_dense)" if dense else
                      "tiled fp32 screen + exact fp64"),
            "kernels": kr, "recall_at_10": rec, "setup_seconds": round(setup, 1),
            "phases_ms_per_step": {key: st[key] / steps for key in
                                   ("join_ms", "join_kernel_ms", "apply_kernel_ms", "reverse_ms",
                                    "assemble_ms", "update_ms", "other_ms")},
        }
        del g, h, u, ds
    return res


def bf_leg(km, ds, device, k=20):
    """Exact k-NN ground truth of the whole config-2 dataset (1M x 1M x 128)
    on the tcgen05 tensor cores (knnm_bf.cuh; exact u8 Gram tiles), host
    numpy output; plus a 200-row spot check against the fp64 SIMT kernel."""
    import torch

    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine(device)
    km.brute_force_graph(ds, km.Metric.L2, k, member_ids=np.arange(8192), device=device)  # warm-up
    torch.cuda.synchronize(device)
    t = time.perf_counter()
    g = km.brute_force_graph(ds, km.Metric.L2, k, device=device)
    torch.cuda.synchronize(device)
    dt = time.perf_counter() - t
    route = eng.bf_route()
    rows = np.sort(np.random.default_rng(0).choice(ds.n, 200, replace=False))
    eng.set_bf_variant(0)
    try:
        eng.begin(np.arange(ds.n, dtype=np.int64), np.zeros(ds.n, dtype=np.int8), k)
        sid, sd = eng.bf_topk(k, rows=rows, exclude_self=True)
    finally:
        eng.set_bf_variant(-1)
    same = bool(np.array_equal(g.ids[rows], sid) and np.array_equal(g.dists[rows], sd))
    n = ds.n
    return {"workload": f"exact {k}-NN graph of the config-2 dataset ({n} x {n} x {ds.d})",
            "route": "tcgen05 kind::i8 (exact u8 Gram tiles)" if route == 1 else "simt fp64",
            "seconds": dt, "pairs_per_s": n * (n - 1) / dt,
            "gram_tops": 2.0 * n * n * ds.d / dt / 1e12,
            "spot_check_rows": 200, "equal_to_fp64_simt": same,
            "note": "host numpy output (240 MB device->host inside the time)"}


def c5_leg(km, device):
    """BASELINE config 5 on one GPU: 8 k=20 subgraphs of 1M points (config-2
    distribution), pairwise S-Merge tree of 3 levels run one after another
    (the 8-GPU placement is tools/c5_tree.py --dist); device-resident,
    CUDA-event time of the three levels."""
    import torch

    from paper_1908_00814_b200.engine import get_engine

    per = 1_000_000
    ds = km.generate_int_gmm(8 * per, 128, 1000, 20.0, seed=7)
    parts = [np.arange(i * per, (i + 1) * per, dtype=np.int64) for i in range(8)]
    graphs = [km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), i + 1, member_ids=p,
                            device=device, out_device=True) for i, p in enumerate(parts)]
    params = km.MergeParams(k=20, seed=3)
    eng = get_engine(device)

    def tree():
        torch.cuda.synchronize(device)
        level, evals, lv = graphs, 0, []
        eng.mark(4)
        while len(level) > 1:
            nxt = []
            for a, b in zip(level[0::2], level[1::2]):
                c = km.DistanceCounter()
                nxt.append(km.s_merge(ds, a, b, params, counter=c, device=device, out_device=True))
                evals += c.count
            eng.mark(5)
            lv.append(eng.elapsed_ms(4, 5) / 1e3 - sum(lv))
            level = nxt
        return evals, lv

    tree()  # warm-up: buffers sized for the 8M-point level
    evals, lv = tree()
    total = sum(lv)
    del graphs
    return {"workload": "config5_tree_8x1M_d128_k20 (levels sequential on one GPU)",
            "seconds": total, "level_seconds": [round(x, 4) for x in lv], "evals": evals,
            "evals_per_s": evals / total}


def tree_leg_dist(km, world, rank, local):
    """BASELINE config 5 across the job's ranks (world = 8: 8 x 1M points,
    one subgraph per GPU; smaller powers of two: the same tree over world x
    1M): distributed.tree_merge, each level's merges sharded over their
    group's GPUs through new_group sub-communicators (NCCL), groups of a
    level concurrent, no re-sharding between levels.  Per-level CUDA-event
    times, max over ranks; a warm-up tree first."""
    import torch
    import torch.distributed as dist

    from paper_1908_00814_b200 import distributed as D
    from paper_1908_00814_b200.engine import get_engine

    per = int(os.environ.get("BENCH_TREE_PER", "1000000"))  # (smaller only in tests)
    ds8 = km.generate_int_gmm(world * per, 128, 1000, 20.0, seed=7)
    sets = [np.arange(r * per, (r + 1) * per, dtype=np.int64) for r in range(world)]
    eng = get_engine(local)
    mine = km.nn_descent(ds8, km.Metric.L2, km.DescentParams(k=20), rank + 1, member_ids=sets[rank],
                         device=local, out_device=True)
    groups = {tuple(m): dist.new_group(m) for _, m in D.tree_groups(world)}

    def group_comm(level, ranks):
        return D.TorchComm(groups[tuple(ranks)]) if rank in ranks else None

    params = km.MergeParams(k=20, seed=3)
    marks = []

    def hook(level, members, cnt):
        torch.cuda.synchronize()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append((level, len(members), ev, cnt.count))

    def run():
        marks.clear()
        torch.cuda.synchronize()
        dist.barrier()
        st = torch.cuda.Event(enable_timing=True)
        st.record()
        D.tree_merge(ds8, {rank: mine}, sets, params, world, group_comm, {rank: eng}, level_hook=hook)
        torch.cuda.synchronize()
        times, evals, prev = [], [], st
        for _, gsize, ev, cnt in marks:
            times.append(prev.elapsed_time(ev) / 1e3)
            evals.append(cnt / gsize)  # summed over ranks: once per group
            prev = ev
        return times, evals

    run()
    times, evals = run()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(times, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e = torch.tensor(evals, dtype=torch.float64, device=dev)
    dist.all_reduce(e, op=dist.ReduceOp.SUM)
    lv = t.tolist()
    total_evals = int(round(sum(e.tolist())))
    return {"workload": f"tree merge of {world} x {per}-point k=20 subgraphs (d=128), one per GPU"
                        + (" = BASELINE config 5" if world == 8 and per == 1_000_000 else ""),
            "seconds": sum(lv), "level_seconds": [round(x, 4) for x in lv], "evals": total_evals,
            "evals_per_s": total_evals / sum(lv), "ranks": world,
            "timing": "per level: CUDA events on each rank, max over ranks (warm-up tree first)"}


def run_b200(args):
    import torch

    world, rank, local = dist_setup()
    # BENCH_BACKEND=gloo (tests of the multi-rank code on one GPU only): all
    # ranks share cuda:0 and the collectives are staged through the host
    test_gloo = os.environ.get("BENCH_BACKEND") == "gloo"
    if test_gloo:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if test_gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        print(f"[bench] rank {dist.get_rank()}/{dist.get_world_size()}: {dist.get_backend()} communicator "
              f"up on cuda:{local} ({torch.cuda.get_device_name(local)})", file=sys.stderr, flush=True)
    rank = int(os.environ.get("RANK", "0"))
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    n = int(CFG["n"] * args.scale)
    k = CFG["k"]
    t_setup = time.perf_counter()
    ds, s1, s2 = make_inputs(km, n)
    eng = get_engine(local)
    if args.join_variant is not None:  # route experiments (default: auto)
        eng.set_join_variant(args.join_variant)
    # subgraphs (untimed), kept resident in HBM as device tensors for `value`
    g_dev = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=k), CFG["g_seed"], member_ids=s1,
                          device=local, out_device=True)
    h_dev = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=k), CFG["h_seed"], member_ids=s2,
                          device=local, out_device=True)

    def to_host(gr):
        out = km.KnnGraph(gr.member_ids, gr.k, gr.metric)
        out.ids = gr.ids.cpu().numpy()
        out.dists = gr.dists.cpu().numpy()
        out.sizes = gr.sizes.cpu().numpy()
        return out

    g_host, h_host = to_host(g_dev), to_host(h_dev)
    # e2e inputs live in page-locked host memory (the contract's "pinned host
    # memory"); outputs are read back into page-locked buffers too
    from paper_1908_00814_b200.engine import pinned_copy

    ds_pinned = km.Dataset.from_dense(pinned_copy(ds.vectors), validate=False)
    for gr in (g_host, h_host):
        gr.ids, gr.dists, gr.sizes = pinned_copy(gr.ids), pinned_copy(gr.dists), pinned_copy(gr.sizes)
    setup_s = time.perf_counter() - t_setup
    params = km.MergeParams(k=k, r=CFG["r"], seed=CFG["merge_seed"])

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    if world > 1:
        # id-sharded merge over the N GPUs (strong scaling: one merge, N ranks)
        from paper_1908_00814_b200 import distributed as D

        comm = D.TorchComm()
        engines = {rank: eng}

        def merge(gg, hh, c, out_device, data=None, p=None):
            return D.s_merge_sharded(data if data is not None else ds, gg, hh, p or params, comm,
                                     engines, counter=c, out_device=out_device)
    else:
        def merge(gg, hh, c, out_device, data=None, p=None):
            return km.s_merge(data if data is not None else ds, gg, hh, p or params, counter=c,
                              device=local, out_device=out_device)

    def step_device():
        c = km.DistanceCounter()
        u = merge(g_dev, h_dev, c, True)
        return c.count, u

    def step_e2e():
        eng.invalidate()  # force the dataset upload inside the timed region
        eng.pinned_outputs = True
        c = km.DistanceCounter()
        u = merge(g_host, h_host, c, False, ds_pinned)
        eng.pinned_outputs = False
        return c.count, u

    # warm-up holds each result until the next step returns, as the timed
    # loop does: the allocator then already caches two sets of output
    # buffers (otherwise the second timed step pays a cudaMalloc)
    u_keep = None
    for _ in range(args.warmup):
        u_keep = step_device()
    del u_keep
    barrier()
    eng.reset_stats()
    eng.set_profiling(True)
    evals = 0
    with ClockSampler(local) as clk:
        torch.cuda.profiler.start()  # ncu --profile-from-start off sees the timed region only
        eng.mark(0)
        step_wall = []
        for _ in range(args.steps):
            t_s = time.perf_counter()
            cnt, u_dev = step_device()
            step_wall.append(round((time.perf_counter() - t_s) * 1e3, 2))
            evals += cnt
        eng.mark(1)
        dev_ms = eng.elapsed_ms(0, 1)
        torch.cuda.profiler.stop()
    barrier()
    st = eng.stats()
    eng.set_profiling(False)
    ms_max = dev_ms
    if world > 1:
        t = torch.tensor([dev_ms], device="cpu" if test_gloo else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max = float(t.item())
    value = evals / (ms_max / 1e3)  # one merge split over the ranks: whole-job rate

    # BASELINE's config-2 sample rate rho = 0.5 (classic NN-Descent sampling;
    # the reference has no rho, so the headline above is rho = 1 = the
    # reference's algorithm bit for bit).  Same inputs, device-resident.
    rho_line = None
    if args.rho_half:
        p_half = km.MergeParams(k=k, r=CFG["r"], seed=CFG["merge_seed"], rho=0.5)
        step_device_half = lambda: merge(g_dev, h_dev, km.DistanceCounter(), True, p=p_half)  # noqa: E731
        # warm-up as for the headline: results held like the timed loop's
        _w = None
        for _ in range(max(2, args.warmup)):
            _w = step_device_half()
        del _w
        barrier()
        eng.reset_stats()
        h_evals, u_half = 0, None
        eng.mark(4)
        for _ in range(args.steps):
            c = km.DistanceCounter()
            u_half = merge(g_dev, h_dev, c, True, p=p_half)
            h_evals += c.count
        eng.mark(5)
        h_ms = eng.elapsed_ms(4, 5)
        if world > 1:
            t = torch.tensor([h_ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            h_ms = float(t.item())
        h_st = eng.stats()
        rho_line = {"rho": 0.5, "ms_per_step": h_ms / args.steps,
                    "merge_seconds": h_ms / args.steps / 1e3,
                    "evals_per_step": h_evals // args.steps,
                    "evals_per_s": h_evals / (h_ms / 1e3),
                    "rounds_per_step": h_st["rounds"] / args.steps,
                    "u_half": u_half}

    # e2e through the public API with host buffers
    _w = step_e2e()  # warm
    del _w
    barrier()
    eng.reset_stats()
    e_evals = 0
    eng.mark(2)
    for _ in range(args.steps):
        cnt, _u = step_e2e()
        e_evals += cnt
        del _u  # release the pinned result before the next step allocates
    eng.mark(3)
    e_ms = eng.elapsed_ms(2, 3)
    est = eng.stats()
    if world > 1:
        t = torch.tensor([e_ms], device="cpu" if test_gloo else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e = e_evals / (e_ms / 1e3)

    # config 5 across the job's GPUs (all ranks take part)
    tree = None
    if (world > 1 and not args.no_c5 and (world & (world - 1)) == 0
            and (args.scale == 1.0 or "BENCH_TREE_PER" in os.environ)):
        try:
            tree = tree_leg_dist(km, world, rank, local)
        except Exception as exc:  # report it; the merge line above stands
            tree = {"error": f"{type(exc).__name__}: {exc}"[:400]}
        eng.set_dataset(ds.vectors, 1)

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    # roofline of the dominant kernel (the local join, timed alone with CUDA
    # events on the engine stream): algorithmic bytes per launch / time.
    # bytes = gathered member rows (sum |M_u| x row bytes: u8 / fp16 rows on
    # the tensor-core route) + hood entries (4 B x members) + written update
    # slots (one packed 8 B record on certified routes, else 8 B dist + 4 B
    # source, per prefilter survivor)
    hbm_peak, peak_kind = peaks()
    inf = eng.info()
    join_kernel = ("k_join_mma<u8>" if inf["cert_u8"] else "k_join_mma<fp16>" if inf["cert_dot"]
                   else "k_join_tiled")
    jk_s = st["join_kernel_ms"] / 1e3
    row_b = st["join_row_bytes"] or 4 * CFG["d"]
    # packed 8-byte slots on the certified routes, f64 + int32 otherwise
    slot_b = 8.0 if (inf["cert"] or inf["cert_dot"]) else 12.0
    join_bytes = (row_b + 4.0) * st["members"] + slot_b * st["written_slots"]
    achieved = join_bytes / jk_s / 1e9 if jk_s > 0 else 0.0
    # SURVEY.md 8(d)'s per-unit figure for the same launches: fp32 member rows
    # (|M_u| * d * 4, the dataset's own format) + 8 B per surviving update.
    # Reported beside the headline, which counts the bytes this kernel
    # actually has to gather (u8 rows on config 2).
    survey_bytes = 4.0 * CFG["d"] * st["members"] + 8.0 * st["written_slots"]
    achieved_survey = survey_bytes / jk_s / 1e9 if jk_s > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_join_traffic.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    u_host = None if args.no_recall else to_host(u_dev)
    rec = recall_sample(ds, u_host, local) if not args.no_recall else None
    if rho_line is not None:
        u_half = rho_line.pop("u_half")
        rho_line["recall_at_10"] = (recall_sample(ds, to_host(u_half), local)
                                    if not args.no_recall else None)
        rho_line["recall_vs_rho1"] = (rho_line["recall_at_10"] - rec
                                      if rec is not None and rho_line["recall_at_10"] is not None else None)
    eng.set_dataset(ds.vectors, 1)
    # join / apply / assembly rooflines of the headline step (same counters)
    kern = kernel_rooflines(st, steps_n := args.steps, CFG["d"], k, slot_b, False, hbm_peak,
                            row_b=row_b)
    kern["assemble"] = {"ms_per_step": st["assemble_ms"] / steps_n,
                        "bytes_per_step": (9.0 * k * st["active_hoods"] + 20.0 * st["members"]) / steps_n}
    a_ms = st["assemble_ms"] / 1e3
    kern["assemble"]["achieved"] = kern["assemble"]["bytes_per_step"] * steps_n / a_ms / 1e9 if a_ms else 0.0
    kern["assemble"].update(peak=hbm_peak, unit="GB/s", frac=kern["assemble"]["achieved"] / hbm_peak,
                            note="phase time (k_mpack_init + k_assemble + scan); bytes: 9k per "
                                 "active hood + 20 B per membership")
    for key in kern:
        kern[key]["share_of_step"] = kern[key]["ms_per_step"] / max(ms_max / steps_n, 1e-9)
    # the bench line's roofline: the dominant kernel of the step (by its own
    # CUDA-event time), with the ncu DRAM traffic of the same kernel
    dom = max(("join", "apply"), key=lambda kk: kern[kk]["ms_per_step"])
    names = {"join": join_kernel, "apply": "k_apply_stream<packed>" if slot_b == 8.0 else "k_apply_stream"}
    models = {"join": f"(row_bytes + 4) * sum|M_u| + {int(slot_b)} * written_slots",
              "apply": "8 * slots read + 13k * (rows loaded + rows stored)"}
    tr = None
    for fn in (f"r2_{dom}_traffic.json",):
        try:
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                tr = json.load(f)
            break
        except Exception:
            pass
    roofline = {"bound": "hbm", "achieved": kern[dom]["achieved"], "peak": hbm_peak, "unit": "GB/s",
                "frac": kern[dom]["frac"], "traffic": tr, "peak_kind": peak_kind,
                "kernel": names[dom], "bytes_model": models[dom],
                "bytes_per_step": kern[dom]["bytes_per_step"],
                "kernel_ms_per_step": kern[dom]["ms_per_step"],
                "kernel_share_of_step": kern[dom]["share_of_step"],
                "join": {"kernel": join_kernel, "achieved": achieved, "frac": achieved / hbm_peak,
                         "traffic": traffic,
                         "survey_formula": {"achieved": achieved_survey, "frac": achieved_survey / hbm_peak,
                                            "bytes_model": "d * 4 * sum|M_u| + 8 * written_slots "
                                                           "(SURVEY 8d: fp32 rows as stored in the dataset)"}}}
    legs = None
    if args.configs and world == 1:
        legs = config_legs(km, args.configs, local, max(1, min(args.steps, 3)), 1, hbm_peak,
                           no_recall=args.no_recall)
        eng.set_dataset(ds.vectors, 1)
    gt = None
    if not args.no_bf and world == 1:
        gt = bf_leg(km, ds, local)
        eng.set_dataset(ds.vectors, 1)
    c5 = None
    if not args.no_c5 and world == 1 and args.scale == 1.0:
        c5 = c5_leg(km, local)
        eng.set_dataset(ds.vectors, 1)
    cpu = None if args.no_cpu else cpu_baseline()
    steps = args.steps
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_max / steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2_smerge_2x500k_d128_k20", "n": n, "d": CFG["d"], "k": k,
                   "r": CFG["r"], "metric": "l2", "rho": 1.0,
                   "parallelism": f"id-sharded x{world} (NCCL all-to-all + all-gather)" if world > 1 else "single",
                   "l2_note": "inputs (512 MB vectors + lists) exceed the 126 MB L2"},
        "merge_seconds": ms_max / steps / 1e3,
        "evals_per_step": evals // steps,
        "recall_at_10": rec,
        "roofline": roofline,
        "stats_per_step": {key: st[key] / steps for key in ("candidates", "written_slots", "exact_evals", "members", "accepted", "join_redos", "rounds")},
        "phases_ms_per_step": {key: st[key] / steps for key in
                               ("join_ms", "join_kernel_ms", "reverse_ms", "assemble_ms", "update_ms", "other_ms")},
        "e2e": {"value": e2e, "unit": UNIT, "ms_per_step": e_ms / steps,
                "h2d_bytes_per_step": est["h2d_bytes"] // steps,
                "d2h_bytes_per_step": est["d2h_bytes"] // steps},
        "kernels": kern,
        "configs": legs,
        "ground_truth": gt,
        "config5": c5 if world == 1 else tree,
        "gpu_launches": st["launches"],
        "step_wall_ms": step_wall,
        "clocks": clk.summary(),
        "setup_seconds": setup_s,
        "cpu_baseline": cpu,
        "rho_0_5": rho_line,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the config size")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-recall", action="store_true")
    ap.add_argument("--join-variant", type=int, default=None,
                    help="force a join route (0 exact, 1 tiled, 2 tensor core)")
    ap.add_argument("--configs", default="c3,c4",
                    help="extra BASELINE config legs at N=1 (comma list; '' to skip)")
    ap.add_argument("--no-bf", action="store_true", help="skip the tensor-core ground-truth leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the config-5 tree leg (one GPU)")
    ap.add_argument("--no-rho-half", action="store_true",
                    help="skip the rho = 0.5 leg (BASELINE's config-2 sample rate)")
    args = ap.parse_args()
    args.rho_half = not args.no_rho_half
    args.configs = [c for c in args.configs.split(",") if c]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        # one process per GPU: re-launch this command under torchrun
        import socket

        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
                  file=sys.stderr, flush=True)
            sys.exit(2)
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
