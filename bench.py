#!/usr/bin/env python
"""Benchmark of the lambda-coupled electrostatics step (one JSON line on rank 0).

A "step" is one pass of the whole hot path (lambda -> charges, pair
list every nstlist, nonbonded + phi, PME spread/FFT/solve/FFT/gather, lambda-group
reduction + bias + lambda/atom BAOAB) for every replica of the rank's batch.

Workload (headline, N=1): BASELINE.json configs[3], the lysozyme-shaped protein (~40k
atoms, 20 lambda-groups incl. 4 multisite His, K = 72), the largest configuration that
fits one GPU, titrated at the 21 pH points of PAPER.md:160 (pH -1 .. 9 step 0.5), all 21
replicas batched in one context.  With N GPUs every rank runs its own 21-replica batch
(weak scaling, replicas only, no collective in the timed region).
`--gpus N` without torchrun starts N ranks itself (torch.distributed.run) and fails when
fewer GPUs exist.

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
DEFAULT_CONFIG = 4
DEFAULT_REPLICAS = {1: 64, 2: 17, 3: 45, 4: 21, 5: 8}
EXTRA = ((2, 17),)                                      # round-1 headline kept as an extra line item


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons polled through NVML every 2 ms during the timed region
    (the recipe's clocks line; nvidia-smi cannot sample a region of a few ms)."""
    BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.max_mhz = None
        self.err = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:          # no NVML: reported as unavailable
            self.err = str(e)
            return self
        self.stop = threading.Event()
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception as e:
                self.err = str(e)
                return
            time.sleep(0.002)

    def __exit__(self, *a):
        if self.err is None:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0,
                    "source": f"NVML ({self.err})"}
        reasons = sorted({k for _, r in self.rows for k, b in self.BITS.items() if r & b})
        return {"sm_mhz": statistics.median(c for c, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 2 ms poll"}


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


# ---------------------------------------------------------------- oracle on the host cores
SAMPLE_CHUNKS = (2, 6)


def _oracle_worker(args):
    """One oracle replica of the workload in its own process: a bounded sample of its step.
    The oracle's real-space sum loops over equal-cost row chunks of 256 atoms (every j is
    tested for each chunk); a step is timed with k1 and k2 chunks and the full step is
    extrapolated linearly to all chunks (every other term of the step runs in full)."""
    cfg, idx, n_steps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle.engine import OracleReplica
    from synthetic.systems import make_system, make_velocities
    s = make_system(cfg)
    pH = s.pH_grid[idx % len(s.pH_grid)]
    k1, k2 = SAMPLE_CHUNKS
    rep = OracleReplica(s, pH, 1 + idx, vel0=make_velocities(s, 1 + idx), params=dict(sample_real_chunks=k1))
    n_chunks = (s.n_atoms + 255) // 256
    out = []
    for _ in range(n_steps):
        rep.p["sample_real_chunks"] = k1
        t0 = time.perf_counter()
        rep.step()
        t1 = time.perf_counter()
        rep.p["sample_real_chunks"] = k2
        rep.step()
        t2 = time.perf_counter()
        per_chunk = max(0.0, ((t2 - t1) - (t1 - t0)) / (k2 - k1))
        out.append((t1 - t0) + (n_chunks - k1) * per_chunk)
    return out


def oracle_throughput(cfg, n_workers, n_steps=1):
    """P concurrent oracle replicas (one process each, single-threaded numpy) -> list of
    extrapolated seconds per full step per replica."""
    import multiprocessing as mp
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(n_workers) as pool:
        res = pool.map(_oracle_worker, [(cfg, k, n_steps) for k in range(n_workers)])
    return [t for r in res for t in r]


def n_oracle_workers():
    n = os.cpu_count() or 1
    if os.environ.get("CPH_REF_WORKERS"):                 # tests: a bounded number of workers
        return max(1, min(n, int(os.environ["CPH_REF_WORKERS"])))
    try:
        import psutil
        n = min(n, max(1, int(psutil.virtual_memory().available / 1.5e9)))    # ~1 GB per worker at C4
    except Exception:
        pass
    return n


def cpu_baseline(cfg, s, R):
    P = n_oracle_workers()
    t0 = time.perf_counter()
    ts = oracle_throughput(cfg, P)
    wall = time.perf_counter() - t0
    per = [DT_PS * 86400.0 / 1000.0 / t for t in ts]                      # ns/day per replica
    return {"value": float(sum(per)), "unit": UNIT, "cores": P, "kind": "oracle",
            "per_core": float(statistics.mean(per)), "aggregate": float(sum(per)),
            "sample": (f"{P} concurrent oracle replicas of {s.name} (one per host core, single-threaded numpy; "
                       f"os.cpu_count() = {os.cpu_count()}), each timing one BAOAB step with {SAMPLE_CHUNKS[0]} and "
                       f"{SAMPLE_CHUNKS[1]} of its {(s.n_atoms + 255) // 256} equal-cost real-space row chunks and "
                       f"extrapolating linearly to the full step (median {statistics.median(ts):.1f} s per full "
                       f"step); value = sum over the P replicas, per_core = mean; {wall:.0f} s wall incl. setup"),
            "gpu_workload_replicas": R}


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle timed on the host cores (rank 0 only), on the same
    workload and metric; each step a bounded sample (see _oracle_worker)."""
    if rank != 0:
        return
    from synthetic.systems import make_system
    cfg = args.config
    s = make_system(cfg)
    R = args.replicas or DEFAULT_REPLICAS[cfg]
    P = n_oracle_workers()
    steps = max(1, min(args.steps, int(os.environ.get("CPH_REF_MAX_STEPS", "3"))))
    t0 = time.perf_counter()
    ts = oracle_throughput(cfg, P, n_steps=steps)
    wall = time.perf_counter() - t0
    per = [DT_PS * 86400.0 / 1000.0 / t for t in ts]
    value = float(sum(per)) / steps                  # P replicas, each timed `steps` times
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": 0, "ms_per_step": 1000.0 * statistics.median(ts), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": s.name, "atoms": s.n_atoms, "replicas_in_sample": P, "replicas_in_workload": R,
                   "pme_grid": list(s.pme_grid), "lambda_coords": s.n_coords},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "oracle",
                         "sample": f"{P} concurrent oracle replicas x {steps} sampled steps ({args.steps} requested; "
                                   f"real-space row chunks {SAMPLE_CHUNKS} extrapolated to the full step); "
                                   f"{wall:.0f} s wall"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU run
def _time_steps(ctx, stream, K, barrier, world):
    import torch
    import torch.distributed as dist
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    ctx.cph_step(K)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def spawn_ranks(args):
    """`--gpus N` without a launcher: re-exec this script under torch.distributed.run."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
        sys.exit(2)
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="cph", choices=["cph", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and args.impl == "cph":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world}", file=sys.stderr)
        sys.exit(2)
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
    # untimed warm-up, rounded up to a whole number of pair-list blocks (nstlist steps, one CUDA
    # graph each): the K timed steps then start on a block boundary and replay the captured
    # graphs instead of launching the partial blocks kernel by kernel; "warmup" reports W as run
    nst = int(s.params["nstlist"])
    W = -(-max(args.warmup, 3) // nst) * nst
    K = args.steps
    ctx.cph_step(W)
    ctx.cph_sync()

    def barrier():
        if world > 1:
            dist.barrier()
    launches0 = ctx.cph_launch_count()
    with ClockSampler(local) as clk:
        ms = _time_steps(ctx, stream, K, barrier, world)
    launches = ctx.cph_launch_count() - launches0
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
    # cuFFT executions are not counted by the library (one R2C and one C2R plan execution per
    # step and replica sub-batch; the sub-batches' launches of a class run side by side)
    S = ctx.sub_batches
    execs = {k: (prof_n[k] if prof_n.get(k) else (S * args.profile_steps if k.startswith("fft") else 0))
             for k in prof_ms}
    per = {k: prof_ms[k] / execs[k] for k in prof_ms if execs[k]}
    total_prof = sum(prof_ms.values())
    kernels = {}
    work = {"nonbonded": ("alu", alg["nonbonded_flop"], "TFLOP/s"), "spread": ("hbm", alg["spread_bytes"], "GB/s"),
            "gather": ("hbm", alg["gather_bytes"], "GB/s"), "solve": ("hbm", alg["solve_bytes"], "GB/s"),
            "fft_r2c": ("hbm", alg["fft_bytes_each"], "GB/s"), "fft_c2r": ("hbm", alg["fft_bytes_each"], "GB/s"),
            "integrate": ("hbm", alg["integrate_bytes"], "GB/s")}
    for k, t_ms in per.items():
        # ms_per_launch: one launch over the whole batch (the S sub-batch launches side by side)
        ent = {"ms_per_launch": t_ms * S, "ms_per_step": prof_ms[k] / args.profile_steps,
               "launches_per_step": execs[k] / args.profile_steps,
               "share_of_step": prof_ms[k] / total_prof if total_prof else None}
        if k in work and t_ms > 0:
            bound, amount, unit = work[k]
            t_ms = prof_ms[k] / args.profile_steps            # the class's device time per step
            if unit == "TFLOP/s":
                ach = amount / (t_ms * 1e-3) / 1e12
                ent.update(bound=bound, achieved=ach, unit=unit, frac=ach / FP32_PEAK_TFLOPS)
            else:
                ach = amount / (t_ms * 1e-3) / 1e9
                ent.update(bound=bound, achieved=ach, unit=unit, frac=ach / hbm)
        if k == "pairlist":
            rebuilds = max(1, args.profile_steps // int(s.params["nstlist"]))
            ent["ms_per_rebuild"] = prof_ms[k] / rebuilds
        kernels[k] = ent
    ours = [k for k in kernels if not k.startswith("fft")]
    dom = max(ours, key=lambda k: prof_ms[k])
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh)
        ent = tr.get("entries", {}).get(f"{s.name}/R{R}", {}).get(dom)
        if ent is not None:
            traffic = ent
            traffic_src = (f"profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per whole-batch launch from "
                           f"one ncu --set full capture ({tr.get('captured', '?')}), not measured in this run")
    except Exception:
        pass
    dk = kernels[dom]
    roof = {"bound": dk.get("bound"), "achieved": dk.get("achieved"),
            "peak": FP32_PEAK_TFLOPS if dk.get("unit") == "TFLOP/s" else hbm, "unit": dk.get("unit"),
            "frac": dk.get("frac"), "traffic": traffic, "traffic_source": traffic_src, "kernel": dom,
            "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz" if dk.get("unit") == "TFLOP/s"
            else f"MEASURED_PEAKS.json hbm_gbs ({hbm_kind})"}

    # whole-step roofline: the pair flops at the FP32 peak plus the spread,
    # gather, two FFTs, solve and integrator bytes at the HBM peak, for all R replicas
    t_roof_ms = 1e3 * (alg["nonbonded_flop"] / (FP32_PEAK_TFLOPS * 1e12) +
                       (alg["spread_bytes"] + alg["gather_bytes"] + 2.0 * alg["fft_bytes_each"] +
                        alg["solve_bytes"] + alg["integrate_bytes"]) / (hbm * 1e9))
    step_roof = {"t_roof_ms": t_roof_ms, "frac": t_roof_ms / ms_step,
                 "definition": "SURVEY 8(d): R x (60 flop x P_rc at the FP32 peak + spread/gather/FFT/solve/"
                               "integrator algorithmic bytes at the HBM peak) / measured ms per step"}

    # e2e through the public API with host buffers: per step, the whole replica state is
    # uploaded from pinned host memory (cph_set_state_all: positions, velocities, lambdas;
    # forces re-evaluated at the uploaded state), one cph_step, and the new state read back
    # (cph_get_state_all).
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

    # titration bookkeeping: gather lambda frames (the run's only collective), fractions
    fr = np.stack([ctx.cph_get_frames(r)[0][:, 0] for r in range(R)])      # lambda_p of group 0
    from paper_2410_01626_b200 import titration
    allf = titration.gather_frames(fr[:, :, None]) if world > 1 else fr[:, :, None]
    ctx.close()

    extra = {}
    if not args.no_extra:
        for c2, r2 in EXTRA:
            s2 = make_system(c2)
            ph2 = np.resize(np.asarray(s2.pH_grid, np.float64), r2)
            x2 = cph.cph_create(s2, ph2, replica_seeds(c2, r2, base=rank), device=local, cuda_stream=stream.cuda_stream,
                                vel_replicas=np.stack([make_velocities(s2, 1000 * rank + r) for r in range(r2)]))
            x2.cph_step(W)
            ms2 = _time_steps(x2, stream, K, barrier, world) / K
            nsd = 1000.0 / ms2 * DT_PS * 86400.0 / 1000.0
            extra[f"{s2.name}/R{r2}"] = {"ms_per_step": ms2, "ns_per_day_per_system": nsd,
                                         "value": nsd * r2 * world, "unit": UNIT}
            x2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, s, R)

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (fp64 lambda reductions and energies)", "data": "synthetic",
        "config": {"workload": s.name, "atoms": s.n_atoms, "replicas_per_gpu": R, "pme_grid": list(s.pme_grid),
                   "lambda_groups": s.n_groups, "lambda_coords": s.n_coords, "pH_points": len(s.pH_grid),
                   "parallelism": f"replicas x{world} (one process per GPU)",
                   "sub_batches": S,
                   "l2": "inputs exceed L2 (no flush): per-step pair-list + grid stream > 126 MB"},
        "ns_per_day_per_system": ns_day_system, "lambda_steps_per_s_per_system": steps_per_s,
        "lambda_coord_updates_per_s": steps_per_s * s.n_coords * R * world,
        "clocks": clocks, "gpu_launches": launches,
        "roofline": roof, "step_roofline": step_roof, "kernels": kernels, "extra": extra,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(blob.size) * world,
                "d2h_bytes_per_step": int(blob.size) * world, "steps": E,
                "path": "cph_set_state_all (pinned H2D + force re-evaluation) + cph_step(1) + cph_get_state_all"},
        "frames_gathered": int(allf.shape[0] * allf.shape[1]),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
