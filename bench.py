#!/usr/bin/env python
"""bench.py — PAM sweeps/s of the B200 iFCTN-TC hot path (arxiv 2511.16358).

One "step" = one PAM sweep (Algorithm 1 lines 2-5): every block (k,i) of the
Gauss–Seidel chain (a2 contraction, a3/a4 Gram/RHS + SPD solves) and the a5 refill, over the
whole synthetic tensor.  Default workload: C5 (64×64×64×64×32 f32, ranks 4, 5% observed,
ρ = 0.1, 50 sweeps configured) — the only HBM-bound config and the one BASELINE.json's
scaling target is quoted on.  X (2.15 GB) is larger than L2, so
no L2 flush is needed between steps.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C5]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the float64 oracle (cpu_baseline / --impl reference) runs one OpenMP thread per physical
# core, packed; read by the OpenMP runtime when the oracle library first runs
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

METRIC = "iFCTN-TC PAM sweeps/s"
UNIT = "sweeps/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def flops_per_sweep(dims, R, N):
    """Declared flop model: 5 flops/entry/block, 11 flops/entry refill, plus the
    small per-block H refresh, Gram/RHS and Cholesky terms."""
    n = float(np.prod(dims))
    f = 0.0
    for k in range(N):
        for i in range(N):
            if i == k:
                continue
            Ik, Ii = dims[k], dims[i]
            f += 5.0 * n + 2 * R * Ii * Ik + (R * (R + 1) + 2 * R) * Ii * Ik + Ik * (R ** 3 / 3 + 2 * R * R)
    return f + 11.0 * n


def bytes_per_sweep(dims, N, s):
    n = float(np.prod(dims))
    return n * (s * N * (N - 1) + 2 * s + 1 / 8)


class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) every 10 ms while running."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index=0):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r) & ~0x1
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.NAMES.items() if self.reasons & k],
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_cpu():
    """(physical cores, CPU model) of this host: unique (package, core) pairs of /proc/cpuinfo
    (psutil's count as a cross-check), the model name line."""
    model, pairs, phys, core = "", set(), None, None
    try:
        for ln in open("/proc/cpuinfo"):
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and not model:
                model = v
            elif k == "physical id":
                phys = v
            elif k == "core id":
                core = v
            elif not k and phys is not None and core is not None:
                pairs.add((phys, core))
                phys = core = None
        if phys is not None and core is not None:
            pairs.add((phys, core))
    except OSError:
        pass
    n = len(pairs)
    if n == 0:
        try:
            import psutil
            n = psutil.cpu_count(logical=False) or 0
        except Exception:
            n = 0
    return max(1, n or (os.cpu_count() or 1)), model


class OracleRun:
    """The float64 oracle (as it stands) on the FULL workload: X⁽⁰⁾ = P_Ω(O), G⁰, then one
    full Algorithm 1 sweep per call (the run continues from sweep to sweep), timed with the
    host clock; one OpenMP thread per physical core, OMP_PROC_BIND=close."""

    def __init__(self, p):
        from oracle import oracle as O
        self.O = O
        self.cores, self.model = host_cpu()
        O.set_threads(self.cores)
        self.p = p
        self.sh = O.Shape(p.dims, p.ranks)
        self.G = p.G0.astype(np.float64)
        self.X = O.init_x(p.observed, p.mask)
        self.F = O.objective(self.sh, self.G, self.X)
        self.done = 0

    def sweep(self):
        t0 = time.perf_counter()
        st, self.F, _ = self.O.sweep(self.sh, self.G, self.X, self.p.mask, self.p.rho, self.F, False)
        el = time.perf_counter() - t0
        if st:
            raise RuntimeError(f"oracle sweep status {st}")
        self.done += 1
        return el

    def sample(self, k, seconds):
        p = self.p
        return (f"{k} full float64 oracle sweep(s) of {p.name} ({'x'.join(map(str, p.dims))}, {p.n} entries, "
                f"all {p.N * (p.N - 1)} blocks + refill, measured, not extrapolated) in {seconds:.1f} s; "
                f"{self.cores} OpenMP threads = physical cores, OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')}; "
                f"CPU: {self.model}")


def oracle_cpu_baseline(p, sweeps=1):
    """cpu_baseline of the bench line: `sweeps` full oracle sweeps of the bench workload."""
    run = OracleRun(p)
    el = sum(run.sweep() for _ in range(sweeps))
    return {"value": sweeps / el, "unit": UNIT, "cores": run.cores, "kind": "oracle",
            "sample": run.sample(sweeps, el), "cpu_model": run.model}


def oracle_single_thread():
    """the float64 oracle on ONE host thread for C1 (its 10 configured sweeps) and
    C2 (one sweep), plus the host CPU model; a baseline, not a target."""
    from oracle import oracle as O
    from synth import make_config
    cpu = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    prev = O.get_threads()
    O.set_threads(1)
    out = {"threads": 1, "cpu_model": cpu, "logical_cpus": os.cpu_count(), "physical_cores": host_cpu()[0]}
    try:
        for name, sweeps in (("C1", 10), ("C2", 1)):
            p = make_config(name)
            sh = O.Shape(p.dims, p.ranks)
            G = p.G0.astype(np.float64)
            X = O.init_x(p.observed, p.mask)
            F = O.objective(sh, G, X)
            t0 = time.perf_counter()
            for _ in range(sweeps):
                st, F, _ = O.sweep(sh, G, X, p.mask, p.rho, F, False)
            el = time.perf_counter() - t0
            out[name] = {"sweeps": sweeps, "seconds": el, "sweeps_per_s": sweeps / el}
    finally:
        O.set_threads(prev)
    return out


def run_reference(args):
    """The base contract's reference arm for this tier: the float64 oracle, as it stands, on
    the host cores — W untimed then K timed FULL sweeps of the bench workload (one step =
    one sweep, the run continuing from step to step).  Rank 0 only under torchrun."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from synth import make_config
    p = make_config(args.config)
    run = OracleRun(p)
    for _ in range(args.warmup):
        run.sweep()
    times = [run.sweep() for _ in range(args.steps)]
    el = sum(times)
    v = args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(p, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": run.cores, "kind": "oracle",
                             "sample": "per step: " + run.sample(1, el / args.steps) +
                                       f"; {args.steps} timed steps after {args.warmup} warm-up sweeps",
                             "cpu_model": run.model},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_seconds": {"min": min(times), "median": statistics.median(times), "max": max(times)}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(p, world):
    return {"workload": p.name, "dims": list(p.dims), "ranks": int(p.ranks.max()),
            "observed_fraction": float(p.mask.mean()), "rho": p.rho,
            "sweeps_configured": p.sweeps, "mask": p.recipe["mask"]["kind"],
            "init": p.recipe["init"]["kind"],
            "l2": "inputs larger than L2 (X = %.2f GB > 126 MB)" % (p.n * p.dtype.itemsize / 1e9)
            if p.n * p.dtype.itemsize > 126e6 else "L2-resident working set (no flush)",
            "parallelism": f"mode-sharded x{world}" if world > 1 else "single GPU"}


def time_sweeps(torch, s, K):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s.sweep(K)
    e1.record()
    torch.cuda.synchronize()
    s.sync()
    return e0.elapsed_time(e1)


def split_profile(prof, N, world, sm):
    """ifctn_profile_sweep's launch order: per block [a2 pass, reduce, (project), solve] with
    the projection only on ranks' blocks k ≠ shard mode; then [refill, finaliser(s)]."""
    k2, red, sol = [], [], []
    t = 0
    for k in range(N):
        for i in range(N):
            if i == k:
                continue
            k2.append(prof[t])
            red.append(prof[t + 1])
            t += 2
            if world > 1 and k != sm:
                sol.append(prof[t] + prof[t + 1])
                t += 2
            else:
                sol.append(prof[t])
                t += 1
    return k2, red, sol, prof[t], sum(prof[t + 1:])


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    tdist = None
    if world > 1:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_16358_b200 import Solver
    from synth import make_config

    p = make_config(args.config)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    N, s_bytes = p.N, p.dtype.itemsize
    R = int(p.ranks.max())
    sm, sb, se = 0, 0, p.dims[0]
    mk_dist = lambda: None
    obs, msk, g0, truth = p.observed, p.mask, p.G0, p.truth
    if world > 1:  # shard X/Ω along the shard mode, the shard-mode chains by column (§8(e))
        from paper_2511_16358_b200 import dist as D
        sm, sb, se = D.shard_range(p.dims, world, rank)
        obs = D.shard_tensor(p.observed, p.dims, sm, sb, se)
        msk = D.shard_tensor(p.mask, p.dims, sm, sb, se)
        truth = D.shard_tensor(p.truth, p.dims, sm, sb, se)
        g0 = D.shard_factors(p.G0, p.dims, p.ranks, sm, sb, se)
        if args.exchange == "peer":  # device-side exchange fused with the solves (peer.cuh)
            ag = D.torch_allgather()
            mk_dist = lambda: D.make_dist(rank, world, -1, peer=True, allgather=ag)
        else:
            uid = D.nccl_unique_id_from_torch()
            mk_dist = lambda: D.make_dist(rank, world, -1, nccl_id=uid)
    obs_d, mask_d, g0_d = dev(obs), dev(msk), dev(g0)

    def barrier():
        if tdist is not None:
            tdist.barrier()
        torch.cuda.synchronize()

    # warm-up on a throwaway context (graph capture, clocks up), then a fresh context so the
    # timed sweeps are sweeps 1..K of the configured run
    warm = Solver(p.dims, p.ranks, obs_d, mask_d, g0_d, rho=p.rho, dist=mk_dist())
    warm.sweep(args.warmup)
    warm.sync()
    prof = warm.profile_sweep()
    warm.close()
    del warm
    s = Solver(p.dims, p.ranks, obs_d, mask_d, g0_d, rho=p.rho, dist=mk_dist())
    barrier()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms = time_sweeps(torch, s, args.steps)
    barrier()
    if tdist is not None:  # the job's time is the slowest rank's
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    launches = s.launch_count()
    rse = s.rse(dev(truth))
    s.close()
    del s
    sweeps_per_s = args.steps / (ms / 1e3)

    # per-kernel split of one sweep (CUDA events on the launching stream)
    k2, red, sol, refill_ms, fin_ms = split_profile(prof, N, world, sm)
    n = int(np.prod(obs.shape)) if world > 1 else p.n  # this rank's entries
    k2_bytes = n * s_bytes                     # algorithmic: X read once per launch
    refill_bytes = n * (2 * s_bytes) + n / 8   # X read + write, 1 mask bit
    hbm, src = peaks()
    k2_gbs = k2_bytes / (statistics.mean(k2) / 1e3) / 1e9
    refill_gbs = refill_bytes / (refill_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(p.name, {}).get("k2_dram_bytes_per_launch")
    except Exception:
        pass

    line = {"metric": METRIC, "value": sweeps_per_s, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32"
            if s_bytes == 4 else "f64", "data": "synthetic", "config": workload_config(p, world),
            "effective_tflops": flops_per_sweep(p.dims, R, N) * sweeps_per_s / 1e12,
            "effective_gbs": bytes_per_sweep(p.dims, N, s_bytes) * sweeps_per_s / 1e9,
            "roofline": {"bound": "hbm", "kernel": "a2 fibre pass (K2)", "achieved": k2_gbs,
                         "peak": hbm, "peak_source": src, "unit": "GB/s", "frac": k2_gbs / hbm,
                         "traffic": traffic,
                         "bytes_per_launch": k2_bytes, "avg_launch_ms": statistics.mean(k2),
                         "launches_per_step": len(k2),
                         # the a2 pass only reads; `peak` is a copy (read + write) peak.  The
                         # measured read-only ceiling of the same data movement (per-warp TMA
                         # ring, scripts/readbw.cu) is 7.18 TB/s on this B200 pool.
                         "read_ceiling_gbs": READ_CEILING_GBS,
                         "frac_of_read_ceiling": k2_gbs / READ_CEILING_GBS},
            "refill": {"achieved": refill_gbs, "frac": refill_gbs / hbm, "ms": refill_ms,
                       "bytes": refill_bytes},
            "a2_ms_by_block": {f"{k},{i}": round(k2[b], 4) for b, (k, i) in enumerate(
                [(k, i) for k in range(N) for i in range(N) if i != k])},
            "kernels_ms_per_sweep": {"a2_pass": sum(k2), "a2_reduce": sum(red),
                                     "a3a4_solve": sum(sol), "a5_refill": refill_ms,
                                     "finalize": fin_ms},
            "gpu_launches": launches, "clocks": clk.summary(), "rse_after_steps": rse}
    if world > 1:
        line["config"]["shard"] = {"mode": sm, "rank0_slice": [sb, se],
                                   "exchange": ("peer memory: each block's solve kernel publishes, waits for and sums "
                                                "the ranks' projected Gram/RHS partials (IFCTN_XCHG_PEER)")
                                   if args.exchange == "peer" else
                                   "NCCL all-reduce of projected Gram/RHS partials per block k != shard mode"}
        line["roofline"]["note"] = "per-rank a2 pass over this rank's shard"

    if not args.no_e2e:
        line["e2e"] = e2e(torch, p, args.steps, obs, msk, g0, mk_dist, barrier, tdist)
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = oracle_cpu_baseline(p)
        if not args.no_extras:
            line["cpu_baseline"]["single_thread"] = oracle_single_thread()
    if not args.no_extras and world == 1:
        line["other_configs"] = other_configs(torch)
        line["rank_grid"] = rank_grid_extra(torch)
        line["mask_gen"] = mask_gen_extra(torch)
        if p.name == "C5":
            line["c5_shard8_rank0"] = shard_rank0_extra(torch, p, 8, k2_gbs)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if tdist is not None:
        tdist.destroy_process_group()
    return 0


def e2e(torch, p, K, obs_h, mask_h, g0_h, mk_dist, barrier, tdist):
    """Same metric through the public API from pinned HOST buffers: ifctn_create copies O,
    Ω and G⁰ host→device, K sweeps each read back their trace row (device→host), and the final
    X is copied back to pinned host memory.  Multi-GPU: each rank its shard; max over ranks."""
    from paper_2511_16358_b200 import IFCTN_X, Solver
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    obs, mask, g0 = pin(obs_h), pin(mask_h), pin(g0_h)
    out = torch.empty(obs.numel(), dtype=torch.float32 if p.dtype == np.float32 else torch.float64).pin_memory()
    res = []
    for it in range(2):
        barrier()
        t0 = time.perf_counter()
        s = Solver(p.dims, p.ranks, obs, mask, g0, rho=p.rho, dist=mk_dist())
        s.sweep(K, trace=True)
        s.reconstruct(IFCTN_X, out=out)
        torch.cuda.synchronize()
        res.append(time.perf_counter() - t0)
        s.close()
        del s
    el = res[-1]
    if tdist is not None:
        t = torch.tensor([el], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        el = float(t.item())
    h2d = obs_h.nbytes + mask_h.nbytes + g0_h.nbytes
    d2h = obs_h.nbytes + K * 40
    return {"value": K / el, "unit": UNIT, "h2d_bytes_per_step": h2d / K,
            "d2h_bytes_per_step": d2h / K, "seconds": el,
            "note": f"one full solve of {K} sweeps per timed iteration (create from pinned host, "
                    "per-sweep trace read, final X to host)"}


def other_configs(torch):
    from paper_2511_16358_b200 import Solver
    from synth import make_config
    out = {}
    for name in ("C1", "C2", "C3", "C4", "C2r"):
        p = make_config(name)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho)
        s.sweep(3)
        s.sync()
        ms = time_sweeps(torch, s, p.sweeps)
        prof = s.profile_sweep()
        rse = s.rse(dev(p.truth))
        met = s.metrics(dev(p.truth))
        s.close()
        sps = p.sweeps / (ms / 1e3)
        out[name] = {"dims": list(p.dims), "dtype": str(p.dtype), "sweeps_timed": p.sweeps,
                     "sweeps_per_s": sps, "us_per_sweep": 1e3 * ms / p.sweeps,
                     "ranks_max": int(p.ranks.max()),
                     "profiled_kernel_us_per_sweep": 1e3 * sum(prof),
                     # launches per block are (a2 pass, reduce, solve): the a3/a4 share
                     "profiled_solve_us_per_sweep": 1e3 * sum(prof[3 * b + 2]
                                                              for b in range(p.N * (p.N - 1))),
                     "effective_gbs": bytes_per_sweep(p.dims, p.N, p.dtype.itemsize) * sps / 1e9,
                     "rse_after_3_plus_timed": rse,
                     "metrics_after_3_plus_timed": {k: (v if v == v and abs(v) != float("inf") else str(v))
                                                    for k, v in met.items()},
                     "regime": "launch/latency-bound" if name == "C1" else "L2-resident"}
    return out


def shard_rank0_extra(torch, p, world, full_k2_gbs):
    """SURVEY §8(e) on one GPU: rank 0's context of the `world`-way C5 run (sharded along
    mode 1 = API mode 0, 8 slices; stored with modes 0 and 1 swapped so fibres stay 64 long),
    one profiled sweep with a no-op host all-reduce (one process).  The a2 pass over the
    268 MB shard against the full tensor's per-pass GB/s."""
    from paper_2511_16358_b200 import Solver
    from paper_2511_16358_b200 import dist as D
    sm, sb, se = D.shard_range(p.dims, world, 0)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    obs = D.shard_tensor(p.observed, p.dims, sm, sb, se)
    d = D.make_dist(0, world, -1, host_allreduce=lambda a: None)
    s = Solver(p.dims, p.ranks, dev(obs), dev(D.shard_tensor(p.mask, p.dims, sm, sb, se)),
               dev(D.shard_factors(p.G0, p.dims, p.ranks, sm, sb, se)), rho=p.rho, dist=d)
    s._dist_keep = d
    s.profile_sweep()
    prof = s.profile_sweep()
    s.close()
    k2, _, _, refill_ms, _ = split_profile(prof, p.N, world, sm)
    n = obs.size
    gbs = n * p.dtype.itemsize / (statistics.mean(k2) / 1e3) / 1e9
    return {"shard_mode": sm, "slice": [sb, se], "entries": n, "a2_ms_mean": statistics.mean(k2),
            "a2_ms_by_block": [round(v, 4) for v in k2], "a2_gbs": gbs,
            "frac_of_full_c5_a2_gbs": gbs / full_k2_gbs,
            "refill_gbs": n * (2 * p.dtype.itemsize + 1 / 8) / (refill_ms / 1e3) / 1e9}


def rank_grid_extra(torch):
    """the paper's two rank-tuning grids through ifctn_grid_run at concurrency
    1 and 8 (wall time of the whole grid, inputs resident, contexts created inside the timed
    region): the MSI grid (P:L485, 18 instances) on the C2 recipe and the traffic grid
    (P:L562, 28 instances) on the Guangzhou-shaped C4 recipe (C4g, 214×61×144)."""
    from synth import MSI_GRID, TRAFFIC_GRID
    return {"msi": _grid_bench(torch, "C2", MSI_GRID,
                               "C2 recipe x MSI rank grid (P:L485): R12 in {3,6,9,15,30,36} x R13=R23 in {3,6,9}"),
            "traffic": _grid_bench(torch, "C4g", TRAFFIC_GRID,
                                   "C4g (214x61x144, C4 recipe) x traffic rank grid (P:L562): "
                                   "R12 in {2,3,4,6,9,12,36} x R13=R23 in {3,6,9,12}")}


def _grid_bench(torch, cfg, pairs, label):
    import time as _t

    from paper_2511_16358_b200.grid import rank_grid
    from synth import grid_rank_matrix, init_factors, make_config
    p = make_config(cfg)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inst = []
    for (r12, r3) in pairs:
        R = grid_rank_matrix(r12, r3)
        g, _ = init_factors(p.dims, R, p.observed, p.mask, p.dtype, "uniform", 0)
        inst.append(dict(ranks=R, rho=p.rho, init=dev(g)))
    obs, mask, truth = dev(p.observed), dev(p.mask), dev(p.truth)
    out = {"workload": label, "instances": len(inst), "sweeps_per_instance": p.sweeps}
    rank_grid(p.dims, obs, mask, inst[:2], 2, truth=truth, concurrency=2)   # warm-up
    for conc in (1, 8):
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        res = rank_grid(p.dims, obs, mask, inst, p.sweeps, truth=truth, concurrency=conc)
        torch.cuda.synchronize()
        el = _t.perf_counter() - t0
        best = min(range(len(res)), key=lambda q: res[q]["rse"])
        out[f"concurrency_{conc}"] = {"seconds": el, "instances_per_s": len(inst) / el,
                                      "sweeps_per_s": len(inst) * p.sweeps / el,
                                      "best_rse": res[best]["rse"], "best_ranks": list(pairs[best])}
    return out


def mask_gen_extra(torch):
    """the on-device RM/FM sampling-set draws (ifctn_mask_uniform / _fibres) at
    C5's RM size and C4's FM size; CUDA events on the current stream, median of 5."""
    from paper_2511_16358_b200 import mask_fibres, mask_uniform
    cases = {"C5_RM": (lambda: mask_uniform(64 ** 4 * 32, 26843546, 0), 64 ** 4 * 32),
             "C4_FM": (lambda: mask_fibres((214, 61, 144, 4), 2, 36551, 0), 214 * 61 * 144 * 4)}
    out = {}
    for name, (fn, n) in cases.items():
        fn()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m = fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            del m
        ms = sorted(ts)[2]
        out[name] = {"n": n, "ms": ms, "entries_per_s": n / (ms * 1e-3)}
    return out


READ_CEILING_GBS = 7180.0   # scripts/readbw.cu: TMA ring, 2 KB stages, 1 CTA/SM


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="multi-GPU exchange: device-side over peer memory (default) or NCCL")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
