#!/usr/bin/env python
"""Benchmark: options priced per second at d=10, N=128, TT rank <= 32.

BASELINE.json's metric is quoted on config 4 (d=10 call-on-min, 129 points
per axis, bond dimension 32).  One *step* prices one batch of ``--batch``
independent config-4-type options per GPU (instance i has parameters drawn
from ``default_rng([4, i])``) through the full hot path:
TT-cross of phi(-z), TT-cross of conj(vhat(z)), tt_inner, prefactor.

  value   device throughput with the option parameters already resident in
          HBM (CUDA events, barrier + synchronize around exactly K steps,
          max over ranks); weak scaling across GPUs.
  e2e     the same metric through the public API with host inputs
          (``price_fourier_tt_batch``): parameter upload and price/report
          download inside the timed region.
  --impl reference
          the reference algorithm on the host CPU cores (the pinned oracle
          port, oracle/ttp_oracle.py -- the reference is pure Python and does
          not travel to the GPU box), one option per core per step.
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

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_ID = 4
METRIC = "options priced/sec at d=10, N=128, TT rank<=32"
UNIT = "options/s"


# ------------------------------------------------------------------ helpers
def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=592,
                    help="options per GPU per step (4 x 148: throughput saturates here, profiles/r01/batch_sweep.json)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="options in the CPU baseline sample (0 = one per core)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spec():
    from paper_2203_02804_b200 import configs
    return configs.CONFIGS[CONFIG_ID]


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(device_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = list(self.rows)
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def alg_work_per_instance(sp, sweeps_phi, sweeps_v):
    """Algorithmic FP64 flops per option (SURVEY.md 8(d) formulas)."""
    from paper_2203_02804_b200.cross import rank_profile
    d, n = sp.d, sp.grid.points_per_axis
    r = rank_profile((n,) * d, sp.bond_dim)
    m_conv = 50_000
    la = 0.0
    for k in range(1, d):
        la += 44.0 * (r[k - 1] * n) * r[k] ** 2           # left-to-right bonds
    conv = 8.0 * m_conv * sum(r[k] * r[k + 1] for k in range(1, d))
    inner = 8.0 * sum(n * (r[k] * r[k] * r[k + 1] + r[k] * r[k + 1] * r[k + 1]) for k in range(d))
    per_sweep = la + conv
    return {"bond_la": la, "conv": conv, "inner": inner,
            "total": per_sweep * (sweeps_phi + sweeps_v) + inner}


# ------------------------------------------------------ CPU reference arm
def _cpu_worker_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:
        pass


def _cpu_price(i):
    from oracle import ttp_oracle as O
    from paper_2203_02804_b200 import configs
    sp = configs.CONFIGS[CONFIG_ID]
    m = configs.make_model(CONFIG_ID, i)
    g = sp.grid
    gm = O.GridModel(m.r, m.sigma, m.T, m.s0, m.strike, m.corr, g.n, g.eta, g.alpha)
    price, _ = O.price_tt(gm, sp.bond_dim, sp.bond_dim, sp.cross_seed, sp.cross_seed)
    return price


def cpu_pool_time(n_opts, procs, start=0):
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs, initializer=_cpu_worker_init) as pool:
        pool.map(_cpu_worker_noop, range(procs))  # spawn + import cost outside the timing
        t0 = time.perf_counter()
        prices = pool.map(_cpu_price, range(start, start + n_opts), chunksize=1)
        wall = time.perf_counter() - t0
    return wall, prices


def _cpu_worker_noop(_):
    import oracle.ttp_oracle  # noqa: F401
    import paper_2203_02804_b200.configs  # noqa: F401
    return 0


def cpu_model_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    per_step = cores
    for w in range(args.warmup):
        cpu_pool_time(per_step, cores, start=0)
    total = 0.0
    for s in range(args.steps):
        wall, _ = cpu_pool_time(per_step, cores, start=0)
        total += wall
    value = per_step * args.steps / total
    sp = spec()
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128/f64",
        "data": "synthetic (seeded default_rng([4, i]) instances, SURVEY.md 8(d))",
        # the GPU arm's workload (same config keys); each reference step is a
        # bounded sample of it (see cpu_baseline.sample)
        "config": {"workload": sp.label + f", batch of {args.batch} independent options per GPU per step",
                   "config_id": CONFIG_ID, "options_per_gpu_per_step": args.batch,
                   "global_batch": args.batch * world, "grid_points_per_axis": sp.grid.points_per_axis,
                   "bond_dim": sp.bond_dim, "parallelism": "host cores (rank 0 only)",
                   "options_timed_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{per_step} config-4 options per step (one per core, 1 BLAS thread "
                                   f"each) on {cpu_model_name()}; the reference is pure Python "
                                   "(no compiled _ref) so its pinned numpy restatement runs"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm
def main():
    args = parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2203_02804_b200 as P
    from paper_2203_02804_b200 import _lib, configs
    from paper_2203_02804_b200.distributed import gather_records, results_to_records, shard_range
    from paper_2203_02804_b200.pricers import run_cross_pair

    sp = spec()
    grid = sp.grid
    shape = (grid.points_per_axis,) * grid.d
    cfg = P.CrossConfig(bond_dim=sp.bond_dim, seed=sp.cross_seed)
    B = args.batch
    n_total = B * world
    lo, hi = shard_range(n_total, rank, world)
    models = [configs.make_model(CONFIG_ID, i) for i in range(lo, hi)]
    prefs = np.array([np.exp(-m.r * m.T) * grid.eta ** grid.d / (2 * np.pi) ** grid.d for m in models])

    # device-resident inputs for the `value` path
    phi_batch = P.OracleBatch([P.PhiGridOracle(m, grid) for m in models])
    v_batch = P.OracleBatch([P.PayoffGridOracle(m, grid, conj=True) for m in models])

    def device_step():
        rp, rv = run_cross_pair(phi_batch, v_batch, shape, cfg, cfg, with_reports=False)
        raw = P.tt_inner_batch(rv.trains, rp.trains)
        return prefs * raw.real, rp, rv

    for _ in range(args.warmup):
        prices, rp, rv = device_step()
    torch.cuda.synchronize()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    clocks = ClockSampler(local)
    _lib.profile_reset()
    _lib.profile_enable(True)
    n0 = _lib.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    t_start.record()
    sweeps_phi = sweeps_v = 0
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 between steps (512 MB > 126 MB L2)
        prices, rp, rv = device_step()
        sweeps_phi += int(rp.counters["sweeps"].sum())
        sweeps_v += int(rv.counters["sweeps"].sum())
        if world > 1:
            recs = np.column_stack([prices, np.zeros((len(prices), 8))])
            gather_records(recs, n_total, device=torch.device("cuda", local))
    t_stop.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed = t_start.elapsed_time(t_stop) / 1e3
    launches = _lib.launch_count() - n0
    _lib.profile_enable(False)
    kstats = _lib.profile_read()
    clk = clocks.stop()
    t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    value = n_total * args.steps / elapsed
    ok = int((rp.status == 0).sum() + (rv.status == 0).sum())

    # e2e through the public API with host inputs
    e2e = None
    if not args.no_e2e:
        for _ in range(1):
            P.price_fourier_tt_batch(models, grid, cfg, cfg, dense_reference="never")
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = P.price_fourier_tt_batch(models, grid, cfg, cfg, dense_reference="never")
            if world > 1:
                gather_records(results_to_records(res), n_total, device=torch.device("cuda", local))
        torch.cuda.synchronize()
        e_el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e_el, op=dist.ReduceOp.MAX)
        d = grid.d
        from paper_2203_02804_b200.cross import _Layout
        lay = _Layout(shape, sp.bond_dim)
        nb = len(models)
        h2d = nb * 8 * ((3 + d + d * d) + 5) + 2 * (lay.set_stride * 4 + 4 * d)
        # prices (complex) + per-instance cross counters of both crosses; the
        # index sets stay on the device until a report's sets are read
        d2h = nb * (16 + 2 * (4 * 5 + 8 * 3) + 8)
        e2e = {"value": n_total * args.steps / float(e_el.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # Roofline of the dominant kernel.  Inside the timed region the phi and
    # vhat crosses run on two streams, so per-launch event durations overlap;
    # one extra untimed step with the two crosses serialized gives clean
    # per-kernel durations (same launches, same inputs) for `achieved`.
    os.environ["TTP_PAIR_STREAMS"] = "0"
    _lib.profile_reset()
    _lib.profile_enable(True)
    device_step()
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    sstats = _lib.profile_read()
    os.environ.pop("TTP_PAIR_STREAMS", None)
    total_serial_ms = sum(v[2] for v in sstats.values())
    dom = max(sstats.items(), key=lambda kv: kv[1][2])
    dom_name, (dom_launch, dom_timed, dom_ms) = dom
    work = alg_work_per_instance(sp, sweeps_phi / max(1, args.steps * B), sweeps_v / max(1, args.steps * B))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "profiles", "fp64_peak.json")))
    except OSError:
        pass
    fp64_peak = peaks.get("fp64_gemm_tflops_8192", 35.4)
    per_kernel_flops = {
        "bond_kernel": work["bond_la"] * (sweeps_phi + sweeps_v) / args.steps,
        "conv_site_kernel": work["conv"] * (sweeps_phi + sweeps_v) / args.steps,
        "tt_inner_kernel": work["inner"] * B,
    }
    traffic = None
    try:
        tr = json.load(open(os.path.join(REPO, "profiles", "ncu_traffic.json")))
        traffic = tr.get(dom_name)
    except OSError:
        pass
    def kernel_roofline(name):
        launches, timed, ms = sstats.get(name, (0, 0, 0.0))
        if name not in per_kernel_flops or not timed:
            return {"bound": "fp64", "kernel": name, "achieved": None, "peak": fp64_peak,
                    "unit": "TFLOP/s", "frac": None, "traffic": None}
        flops_per_launch = per_kernel_flops[name] / max(1, launches)
        achieved = flops_per_launch / (ms / timed / 1e3) / 1e12
        t_launch, t_timed, t_ms = kstats.get(name, (0, 0, 0.0))
        return {"bound": "fp64", "kernel": name, "achieved": achieved, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": achieved / fp64_peak, "traffic": traffic if name == dom_name else None,
                "peak_source": "profiles/fp64_peak.json (cuBLAS DGEMM 8192^3 on this pool's B200)",
                "avg_launch_ms": ms / timed, "alg_flops_per_launch": flops_per_launch,
                "share_of_step": ms / total_serial_ms if total_serial_ms else None,
                "avg_launch_ms_timed_region": (t_ms / t_timed) if t_timed else None}

    roofline = kernel_roofline(dom_name)
    roofline["note"] = ("durations from one untimed, stream-serialized step (the timed region overlaps the "
                        "phi and vhat crosses on two streams); algorithmic flops per SURVEY.md 8(d)")
    # the bond kernel is memory bound: its measured DRAM traffic (ncu, same
    # batch) per event-timed launch, against the measured HBM copy peak
    try:
        hbm_peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except (OSError, ValueError):
        hbm_peak = None
    if traffic and roofline.get("avg_launch_ms") and hbm_peak:
        rate = traffic / (roofline["avg_launch_ms"] / 1e3) / 1e9
        roofline["dram"] = {"bytes_per_launch": traffic, "achieved_gbs": rate, "peak_gbs": hbm_peak,
                            "frac": rate / hbm_peak,
                            "source": "profiles/ncu_traffic.json (dram__bytes_read+write, ncu --set full, "
                                      "same batch) / avg_launch_ms; MEASURED_PEAKS.json hbm_gbs"}
    secondary = [kernel_roofline(k) for k in ("conv_site_kernel", "tt_inner_kernel") if k != dom_name]

    cpu_baseline = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        n_opts = args.cpu_sample or cores
        wall, cpu_prices = cpu_pool_time(n_opts, cores, start=0)
        cpu_baseline = {"value": n_opts / wall, "unit": UNIT, "cores": min(cores, n_opts), "kind": "port",
                        "sample": f"{n_opts} config-4 options (instances 0..{n_opts - 1}) on {cpu_model_name()}, "
                                  "pinned numpy restatement of the reference, 1 BLAS thread per process",
                        "wall_s": wall}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128/f64",
        "data": "synthetic (seeded default_rng([4, i]) config-4 instances, SURVEY.md 8(d))",
        "config": {"workload": sp.label + f", batch of {B} independent options per GPU per step",
                   "config_id": CONFIG_ID, "options_per_gpu_per_step": B, "global_batch": n_total,
                   "grid_points_per_axis": grid.points_per_axis, "bond_dim": sp.bond_dim,
                   "parallelism": f"instance-sharded dp{world}",
                   "l2": "512 MB L2 flush before every timed step; per-step working set ~GBs >> 126 MB L2",
                   "sweeps_per_option": [sweeps_phi / (args.steps * B), sweeps_v / (args.steps * B)],
                   "instances_ok": ok},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roofline,
        "roofline_secondary": secondary,
        "cpu_baseline": cpu_baseline,
        "clocks": clk,
        "kernels": {k: {"launches": v[0], "ms": v[2]} for k, v in kstats.items() if v[0]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
