#!/usr/bin/env python
"""Benchmark of the lambda-coupled electrostatics step (one JSON line on rank 0).

A "step" is one pass of the whole hot path (lambda -> charges, pair
list every nstlist, nonbonded + phi, PME spread/FFT/solve/FFT/gather, lambda-group
reduction + bias + lambda/atom BAOAB) for every replica of the rank's batch.

Workload (BASELINE.json configs[1]): the GEAHG-shaped pentapeptide system (~7k atoms,
Glu 2-state + His 3-state lambda-groups) titrated at the paper's 17 pH points
(PAPER.md:22), all 17 replicas batched in one context on one GPU.  With N GPUs every
rank runs its own 17-replica batch (weak scaling, replicas only, no collective in the
timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cph|reference] [--config 1..5]
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ns/day & λ-steps/s per system at 1 B200; pH-replica throughput at 2/4/8 GPUs"
UNIT = "ns/day (summed over pH replicas)"
DT_PS = 0.002
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12      # SMs x FP32 lanes x FMA x max clock
DEFAULT_REPLICAS = {1: 64, 2: 17, 3: 45, 4: 20, 5: 1}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic(sys_, R):
    """Per-launch algorithmic work for R replicas."""
    N = sys_.n_atoms
    V = float(np.prod(sys_.box))
    rho = N / V
    rc = sys_.params["rc"]
    p_rc = N * rho * 4.0 / 3.0 * math.pi * rc ** 3 / 2.0
    K = sys_.pme_grid
    K3 = K[0] * K[1] * K[2]
    Kc = K[0] * K[1] * (K[2] // 2 + 1)
    return {
        "pairs_rc": p_rc * R,
        "nonbonded_flop": 60.0 * p_rc * R,
        "spread_bytes": (16.0 * N + 4.0 * K3) * R,
        "gather_bytes": (32.0 * N + 4.0 * K3) * R,
        "solve_bytes": 16.0 * Kc * R,
        "fft_bytes_each": (4.0 * K3 + 8.0 * Kc) * R,
        "integrate_bytes": 96.0 * N * R,
    }


def cpu_baseline(cfg, budget_s=20.0):
    """The oracle as it stands, one replica of the same workload, on the host cores."""
    from oracle.engine import OracleReplica
    from synthetic.systems import make_system, make_velocities
    s = make_system(cfg)
    rep = OracleReplica(s, s.pH_grid[0], 1, vel0=make_velocities(s, 1))
    t0 = time.perf_counter()
    n = 0
    while True:
        rep.step()
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    t = time.perf_counter() - t0
    return n, t


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from synthetic.systems import make_system
    cfg = args.config
    s = make_system(cfg)
    R = args.replicas or DEFAULT_REPLICAS[cfg]
    budget = float(os.environ.get("CPH_REF_BUDGET_S", "150"))
    from oracle.engine import OracleReplica
    from synthetic.systems import make_velocities
    rep = OracleReplica(s, s.pH_grid[0], 1, vel0=make_velocities(s, 1))
    if args.warmup:
        rep.step()
    t0 = time.perf_counter()
    n = 0
    while n < args.steps:
        rep.step()
        n += 1
        if time.perf_counter() - t0 > budget:
            break
    t = time.perf_counter() - t0
    steps_per_s = n / t
    value = steps_per_s * DT_PS * 86400.0 / 1000.0          # one replica on the host
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": n, "warmup": min(args.warmup, 1), "ms_per_step": 1000.0 * t / n, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": s.name, "atoms": s.n_atoms, "replicas_in_sample": 1, "replicas_in_workload": R,
                   "pme_grid": list(s.pme_grid), "lambda_coords": s.n_coords},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{n} of {args.steps} requested oracle steps of 1 of {R} replicas "
                                   f"(per-step cost is constant; bounded to {budget:.0f} s)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="cph", choices=["cph", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2410_01626_b200 as cph
    from synthetic.systems import make_system, make_velocities, replica_seeds
    cfg = args.config
    s = make_system(cfg)
    R = args.replicas or DEFAULT_REPLICAS[cfg]
    pH = np.resize(np.asarray(s.pH_grid, np.float64), R)
    seeds = replica_seeds(cfg, R, base=rank)
    vel = np.stack([make_velocities(s, 1000 * rank + r) for r in range(R)])
    # a dedicated (non-default) torch stream: the library launches on it and the CUDA
    # events below are recorded on it
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx = cph.cph_create(s, pH, seeds, vel_replicas=vel, device=local, cuda_stream=stream.cuda_stream)
    W = max(args.warmup, 3)
    K = args.steps
    ctx.cph_step(W)
    ctx.cph_sync()

    def barrier():
        if world > 1:
            dist.barrier()
    launches0 = ctx.cph_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        ctx.cph_step(K)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = ctx.cph_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ctx.cph_sync()
    ms_step = ms / K
    steps_per_s = 1000.0 / ms_step
    ns_day_system = steps_per_s * DT_PS * 86400.0 / 1000.0
    value = ns_day_system * R * world

    # per-kernel live timing (CUDA events on the launching stream, serialised)
    prof_ms, prof_n = ctx.cph_profile_steps(args.profile_steps)
    ctx.cph_sync()
    alg = algorithmic(s, R)
    hbm, hbm_kind = peaks()
    per = {k: (prof_ms[k] / prof_n[k] if prof_n.get(k) else (prof_ms[k] / args.profile_steps)) for k in prof_ms}
    total_prof = sum(prof_ms.values())
    kernels = {}
    work = {"nonbonded": ("alu", alg["nonbonded_flop"], "TFLOP/s"), "spread": ("hbm", alg["spread_bytes"], "GB/s"),
            "gather": ("hbm", alg["gather_bytes"], "GB/s"), "solve": ("hbm", alg["solve_bytes"], "GB/s"),
            "fft_r2c": ("hbm", alg["fft_bytes_each"], "GB/s"), "fft_c2r": ("hbm", alg["fft_bytes_each"], "GB/s"),
            "integrate": ("hbm", alg["integrate_bytes"], "GB/s")}
    for k, t_ms in per.items():
        ent = {"ms_per_launch": t_ms, "share_of_step": prof_ms[k] / total_prof if total_prof else None}
        if k in work and t_ms > 0:
            bound, amount, unit = work[k]
            if unit == "TFLOP/s":
                ach = amount / (t_ms * 1e-3) / 1e12
                ent.update(bound=bound, achieved=ach, unit=unit, frac=ach / FP32_PEAK_TFLOPS)
            else:
                ach = amount / (t_ms * 1e-3) / 1e9
                ent.update(bound=bound, achieved=ach, unit=unit, frac=ach / hbm)
        kernels[k] = ent
    ours = [k for k in per if not k.startswith("fft")]
    dom = max(ours, key=lambda k: prof_ms[k])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get(f"{s.name}/R{R}", {}).get(dom)
    except Exception:
        pass
    dk = kernels[dom]
    roof = {"bound": dk.get("bound"), "achieved": dk.get("achieved"),
            "peak": FP32_PEAK_TFLOPS if dk.get("unit") == "TFLOP/s" else hbm, "unit": dk.get("unit"),
            "frac": dk.get("frac"), "traffic": traffic, "kernel": dom,
            "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz" if dk.get("unit") == "TFLOP/s"
            else f"MEASURED_PEAKS.json hbm_gbs ({hbm_kind})"}

    # e2e through the public API with host buffers: per step, the whole replica state is
    # uploaded from pinned host memory (cph_set_state_all, which re-evaluates forces), one
    # cph_step, and the new state read back (cph_get_state_all).
    blob = ctx.cph_get_state_all()
    pinned_in = torch.from_numpy(blob.copy()).pin_memory().numpy()
    pinned_out = torch.empty(blob.size, dtype=torch.uint8).pin_memory().numpy()
    E = max(1, args.e2e_steps)
    ctx.cph_set_state_all(pinned_in)
    ctx.cph_step(1)
    ctx.cph_get_state_all(pinned_out)
    barrier()
    t0 = time.perf_counter()
    for _ in range(E):
        ctx.cph_set_state_all(pinned_in)
        ctx.cph_step(1)
        ctx.cph_get_state_all(pinned_out)
    t_e2e = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([t_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e_value = (E / t_e2e) * DT_PS * 86400.0 / 1000.0 * R * world

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n, t = cpu_baseline(cfg)
        cpu = {"value": n / t * DT_PS * 86400.0 / 1000.0, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{n} oracle steps of 1 replica of {s.name} ({t:.1f} s)"}

    # titration bookkeeping: gather lambda frames (the run's only collective), fractions
    fr = np.stack([ctx.cph_get_frames(r)[0][:, 0] for r in range(R)])      # lambda_p of group 0
    from paper_2410_01626_b200 import titration
    allf = titration.gather_frames(fr[:, :, None]) if world > 1 else fr[:, :, None]

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (fp64 lambda reductions and energies)", "data": "synthetic",
        "config": {"workload": s.name, "atoms": s.n_atoms, "replicas_per_gpu": R, "pme_grid": list(s.pme_grid),
                   "lambda_groups": s.n_groups, "lambda_coords": s.n_coords, "pH_points": len(s.pH_grid),
                   "parallelism": f"replicas x{world} (one process per GPU)",
                   "l2": "inputs exceed L2 (no flush): per-step neighbour-list stream %.0f MB > 126 MB"
                         % (2.0 * alg["pairs_rc"] * 1.331 * 4 / 1e6)},
        "ns_per_day_per_system": ns_day_system, "lambda_steps_per_s_per_system": steps_per_s,
        "lambda_coord_updates_per_s": steps_per_s * s.n_coords * R * world,
        "clocks": clocks, "gpu_launches": launches,
        "roofline": roof, "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(blob.size) * world,
                "d2h_bytes_per_step": int(blob.size) * world, "steps": E,
                "path": "cph_set_state_all (pinned H2D + force re-evaluation) + cph_step(1) + cph_get_state_all"},
        "frames_gathered": int(allf.shape[0] * allf.shape[1]),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
