"""Benchmark: monodomain DoF*steps/s of config 2 (BASELINE.json configs[2]).

One "step" = one IMEX-BDF2 monodomain time step (TissueSolver.step,
reference simulation.py:425-483) of the 20x7x3 mm TTP06 slab at h=0.1 mm
(442,401 nodes): fused ionic update + RHS + Jacobi PCG + activation.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* ours: warm-up W steps from rest, then K timed steps (the propagation phase:
  the stimulus fires at t=0, CG needs 7..18 iterations per step).  `value` is
  device-timed (CUDA events, barrier + synchronize both sides, max over
  ranks) with all state resident in HBM; `e2e` goes through the public API
  with host buffers: the initial state is uploaded from a host checkpoint
  payload in pinned memory (TissueSolver.restore) inside the timed region,
  and every step
  reads back the run() output row (t, u_min, u_max, 9 probes) to the host.
* reference: the reference algorithm on the host CPU cores (oracle port,
  oracle/, pinned bit-identical to the reference; the reference itself is
  Python+numba and cannot travel to the GPU box) on a bounded sample of the
  same workload.

The ionic state ring (4 x 18 x 442,401 doubles = 255 MB) exceeds the 126 MB
L2, so no explicit L2 flush is done between steps.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "monodomain DoF*steps/s (config 2: TTP06 slab 442,401 nodes, BDF2, Jacobi PCG)"
UNIT = "DoF*steps/s"
FALLBACK_HBM = 6650.0


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"],
                    "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def traffic_of(kernel):
    """ncu figures of one launch of `kernel` from the committed capture
    (profiles/ncu_traffic.json, written by scripts/summarize_ncu.py):
    {"dram_bytes", "fp64_flops", ...}, or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        for k, v in d.items():
            if kernel in k:
                return v if isinstance(v, dict) else {"dram_bytes": v}
    return None


def fp64_peak_tflops():
    """FP64 FMA peak: profiles/fp64_peak.json (scripts/fp64_peak.cu run on the
    box), else the nominal 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz."""
    p = ROOT / "profiles" / "fp64_peak.json"
    if p.exists():
        return float(json.loads(p.read_text())["fp64_tflops"]), "measured"
    return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


PLATEAU_STEP = 2500          # t = 50 ms at dt = 2e-5 s: every node depolarised


def cpu_sample(steps, threads=None, warmup=2):
    """Oracle port of the reference step on cfg 2: `warmup` (>= 2, the BDF
    start-up) untimed steps from rest, then `steps` timed steps."""
    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs

    ns = configs.this_package()
    cfg = configs.config2(ns)
    orc = O.OracleTissue(cfg)
    for _ in range(max(2, warmup)):   # BDF1 then BDF2 systems built
        orc.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.step()
    wall = time.perf_counter() - t0
    n = cfg.mesh.nodes.shape[0]
    return n * steps / wall, wall, O.num_threads(), orc.iters[max(2, warmup):]


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # K timed steps of the workload after W warm-up steps, like our arm
    w = max(2, args.warmup)
    value, wall, cores, its = cpu_sample(args.steps, warmup=w)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": w,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2 TTP06 slab 20x7x3 mm h=0.1 mm, BDF2, dt=2e-5 s",
                   "nodes": 442401},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"steps {w + 1}..{w + args.steps} of config 2 from rest "
                                   f"(CG iterations {min(its)}..{max(its)}), full mesh"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    # MDX_BENCH_DIST=1: the distributed solver even at one rank (tests the N > 1 path on one GPU)
    use_dist = world > 1 or os.environ.get("MDX_BENCH_DIST") == "1"
    if use_dist:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    ns = configs.this_package()
    cfg = configs.config2(ns)
    n = cfg.mesh.nodes.shape[0]
    if use_dist:
        return run_distributed(args, cfg, n, rank, world, local, dist)
    solver = TissueSolver(cfg)
    init_payload = solver.checkpoint_payload()   # host copy of the initial state
    for _ in range(args.warmup):
        solver.enqueue_step()
    solver.sync()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-timed region ------------------------------------------------
    ev_ionic = []
    launches0 = solver.launches
    barrier()
    with ClockSampler(local) as clocks:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record()
            solver.enqueue_step(events=(e1, e2))
            ev_ionic.append((e0, e1, e2))
        end.record()
        barrier()
    launches = solver.launches - launches0
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ionic_ms = np.array([a.elapsed_time(b) for a, b, _ in ev_ionic])
    solve_ms = np.array([b.elapsed_time(c) for _, b, c in ev_ionic])
    its = solver.iterations_log()[-args.steps:]
    solver.sync()

    # ---- plateau phase (reported beside the headline) ------------------------
    # the propagation phase is CG-bound, the plateau (every node
    # depolarised, CG 1-2 iterations) ionic/FP64-bound.  The same solver is
    # advanced untimed to t = 50 ms, then K steps are device-timed again.
    plateau = None
    if world == 1 and not args.no_plateau:
        while solver.step_index < PLATEAU_STEP:
            solver.enqueue_step()
        solver.sync()
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        barrier()
        p0.record()
        for _ in range(args.steps):
            solver.enqueue_step()
        p1.record()
        barrier()
        pms = p0.elapsed_time(p1)
        pits = solver.iterations_log()[-args.steps:]
        solver.sync()
        plateau = {"value": n * args.steps / (pms * 1e-3), "unit": UNIT,
                   "ms_per_step": pms / args.steps, "from_step": PLATEAU_STEP,
                   "cg_iters_per_step": [int(pits.min()), float(pits.mean()), int(pits.max())],
                   "bytes_per_step_frac_hbm": float(
                       n * (562 + 104 * pits.astype(np.float64)).sum()
                       / (pms * 1e-3) / 1e9 / peaks()[0])}

    # ---- end-to-end through the public API ----------------------------------
    e2e_solver = TissueSolver(cfg)
    probes = [ns.nearest_node(cfg.mesh, p) for p in configs.corner_probes()]
    probes.append(ns.nearest_node(cfg.mesh, (10e-3, 3.5e-3, 1.5e-3)))
    pidx = torch.tensor(probes, device="cuda")
    e2e_steps = args.steps + args.warmup
    # the host input: the initial-state checkpoint in pinned memory
    payload_pinned = torch.frombuffer(bytearray(init_payload), dtype=torch.uint8).pin_memory()
    pinned = torch.empty((e2e_steps, 2 + len(probes)), dtype=torch.float64, pin_memory=True)
    barrier()
    t0 = time.perf_counter()
    e2e_solver.restore(payload_pinned)
    for k in range(e2e_steps):
        # the run() output row of every step, written by the solve into pinned host memory
        e2e_solver.enqueue_step(record=(pidx, pinned[k]))
    e2e_solver.sync()
    barrier()
    assert np.isfinite(pinned.numpy()).all()
    e2e_wall = time.perf_counter() - t0
    e2e_value = n * e2e_steps * world / e2e_wall

    hbm, peak_kind = peaks()
    fp64_peak, fp64_kind = fp64_peak_tflops()
    nv = 18
    steps_k = its.astype(np.float64)
    # SURVEY.md 8(d) algorithmic bytes per node-step (fp64, BDF2, fused design):
    #   ionic update 8*(3nv+3) = 456 (read u_n, u_n-1, W_n, W_n-1; write W_n+1, c)
    #   PCG launch: RHS 16 + CG setup 56 + activation 34 + 104 per CG iteration
    #   whole step 562 + 104 k, k = this step's CG iterations
    ionic_bytes = n * 8 * (3 * nv + 3)
    pcg_bytes = n * (16 + 56 + 34 + 104 * steps_k)
    step_bytes = n * (562 + 104 * steps_k)
    pcg_share = float(solve_ms.sum() / (ionic_ms.sum() + solve_ms.sum()))
    ionic_avg = float(ionic_ms.mean()) * 1e-3
    achieved = ionic_bytes / ionic_avg / 1e9
    pcg_achieved = float(pcg_bytes.sum() / (solve_ms.sum() * 1e-3) / 1e9)
    step_achieved = float(step_bytes.sum() / (ms * 1e-3) / 1e9)
    dominant_pcg = pcg_share > 0.5
    t_ionic = traffic_of("tissue_ionic")
    roof_ionic = {"bound": "hbm", "kernel": "tissue_ionic<TTP06,2>",
                  "achieved": achieved, "peak": hbm, "peak_kind": peak_kind,
                  "unit": "GB/s", "frac": achieved / hbm,
                  "bytes_per_launch": ionic_bytes,
                  "traffic": t_ionic.get("dram_bytes") if t_ionic else None}
    if t_ionic and t_ionic.get("fp64_flops"):
        # FP64 flops per cell from the ncu SASS counts of one launch (per-cell
        # constant up to branch divergence), scaled to this launch's n
        flops = t_ionic["fp64_flops"] / t_ionic.get("n", n) * n
        roof_ionic["fp64"] = {"achieved": flops / ionic_avg / 1e12, "peak": fp64_peak,
                              "peak_kind": fp64_kind, "unit": "TFLOP/s",
                              "frac": flops / ionic_avg / 1e12 / fp64_peak,
                              "flops_per_launch": flops}
    t_pcg = traffic_of("pcg_resident_kernel") or traffic_of("pcg_kernel")
    roof_pcg = {"bound": "hbm", "kernel": "pcg_resident_kernel<tissue,4> (vectors in SMEM: "
                "HBM roofline of the unfused algorithm's bytes)",
                "achieved": pcg_achieved, "peak": hbm, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": pcg_achieved / hbm,
                "bytes_per_launch": float(pcg_bytes.mean()),
                "traffic": t_pcg.get("dram_bytes") if t_pcg else None}
    roof_step = {"bound": "hbm", "achieved": step_achieved, "peak": hbm, "unit": "GB/s",
                 "frac": step_achieved / hbm, "bytes_per_step": float(step_bytes.mean()),
                 "formula": "n*(562 + 104*k) per step (SURVEY.md 8(d))"}
    line = {
        "metric": METRIC, "value": n * args.steps * world / (ms * 1e-3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2 TTP06 slab 20x7x3 mm h=0.1 mm (442,401 nodes), "
                               "BDF2, dt=2e-5 s, steps from rest (propagation phase)",
                   "operator": {1: "stencil27 class tables", 2: "csr", 3: "sell32"}[solver.op.kind],
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "state ring 255 MB > L2; no flush",
                   "cg_iters_per_step": [int(its.min()), float(its.mean()), int(its.max())]},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
        "kernels": {"ionic_ms": float(ionic_ms.mean()), "pcg_ms": float(solve_ms.mean()),
                    "pcg_share": pcg_share},
        "roofline": roof_pcg if dominant_pcg else roof_ionic,
        "roofline_other": roof_ionic if dominant_pcg else roof_pcg,
        "roofline_step": roof_step,
        "phases": {"propagation": {"value": n * args.steps * world / (ms * 1e-3),
                                   "from_step": args.warmup},
                   "plateau": plateau},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": len(init_payload) / e2e_steps,
                "d2h_bytes_per_step": 8 * (2 + len(probes))},
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        value, wall, cores, cits = cpu_sample(args.cpu_steps)
        line["cpu_baseline"] = {
            "value": value, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"oracle port, steps 3..{2 + args.cpu_steps} of config 2 from rest"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_distributed(args, cfg, n, rank, world, local, dist):
    """N > 1: config 2 split over the ranks (z-slabs, NCCL halo + all-reduce),
    strong scaling (total work fixed)."""
    import torch

    from paper_2308_01651_b200.distributed import DistributedTissueSolver

    solver = DistributedTissueSolver(cfg)
    for _ in range(args.warmup):
        solver.step()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = solver.launches
    with ClockSampler(local) as clocks:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(args.steps):
            solver.step()
        end.record()
        dist.barrier()
        torch.cuda.synchronize()
    t = torch.tensor([start.elapsed_time(end)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    its = np.array(solver.iters[-args.steps:])
    launches = solver.launches - launches0

    # ---- e2e: every rank re-uploads its slab state (rings, activation) from
    # pinned host memory, then runs the same K steps through the public
    # step() and reads each step's local potential range back to the host
    names = ("u_ring", "w_ring", "act_time", "best_slope", "frozen")
    snap = {k: getattr(solver, k).cpu().pin_memory() for k in names}
    head, step_index, time_s = solver.head, solver.step_index, solver.time
    h2d = sum(v.numel() * v.element_size() for v in snap.values())
    sl = solver.slab
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in names:
        getattr(solver, k).copy_(snap[k], non_blocking=True)
    solver.head, solver.step_index, solver.time = head, step_index, time_s
    for _ in range(args.steps):
        solver.step()
        u = solver.potential_local()[sl.own_begin:sl.own_end]
        torch.stack([u.min(), u.max()]).cpu()
    dist.barrier()
    torch.cuda.synchronize()
    wall = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    e2e = {"value": n * args.steps / float(wall.item()), "unit": UNIT,
           "h2d_bytes_per_step": h2d * world / args.steps, "d2h_bytes_per_step": 16 * world}
    if rank == 0:
        line = {
            "metric": METRIC, "value": n * args.steps / (ms * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2 TTP06 slab 442,401 nodes, BDF2, dt=2e-5 s",
                       "parallelism": f"z-slab domain decomposition x{world}, NCCL halo + "
                                      "all-reduce, pipelined PCG with device-resident scalars, "
                                      "halo overlapped with the interior-plane sweep",
                       "cg_iters_per_step": [int(its.min()), float(its.mean()),
                                             int(its.max())]},
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--no-plateau", action="store_true",
                    help="skip the plateau-phase sample (t = 50 ms) of the same run")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=12)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
