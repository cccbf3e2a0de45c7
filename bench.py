"""Benchmark: monodomain DoF*steps/s on config 4 (BASELINE.json configs[4]).

One "step" = one IMEX-BDF2 monodomain time step (TissueSolver.step,
reference simulation.py:425-483): ionic update (TTP06, three volumes with
duplicated interface states), ICI right-hand side, Jacobi PCG of
(alpha/dt M + K) u = b to rtol 1e-10, activation map.

Headline workload: the config-4 ventricle - truncated prolate-spheroid shell,
P1 tets, 10,276,240 nodes / 59,904,000 tets, helix fibers, endo/mid/epi
volumes, apical stimulus - the largest BASELINE mesh that fits one GPU.
The timed window starts at step 500 (t = 10 ms: the activation front is
travelling through the wall, 61-99 CG iterations per step), reached by
untimed stepping from rest; W warm-up steps precede it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg4|cfg2]

* ours: `value` is device-timed (CUDA events on the launch stream, barrier +
  synchronize both sides, max over ranks) with all state resident in HBM;
  `e2e` goes through the public API with host buffers: the window's start
  state is uploaded from a checkpoint payload in pinned host memory (the
  reference's format with the history levels a restart of this BDF order
  reads; TissueSolver.restore) inside the timed region, then the same K steps run
  and each writes its run() output row (u_min, u_max, 9 probes) into pinned
  host memory.  `secondary` is config 2 (442,401-node TTP06 slab) from step
  250 (t = 5 ms, mid-propagation).
* reference: the reference algorithm on the host CPU cores (oracle port in
  oracle/, pinned bit-identical to the reference package, which is
  Python+numba and not installable on the GPU box) on the same mesh: the
  BDF start-up steps from rest untimed, then K' <= K timed steps (bounded to
  ~a minute of CPU work).

The ionic state ring (2 x 18 x 10.8 M doubles = 3.1 GB) and the operator
(6 x 82 MB) exceed the 126 MB L2 many times over: no explicit L2 flush.
"""

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

UNIT = "DoF*steps/s"
FALLBACK_HBM = 6650.0

WORKLOADS = {
    "cfg4": dict(
        metric="monodomain DoF*steps/s (config 4: prolate-spheroid ventricle, P1 tets, "
               "10,276,240 nodes, TTP06 x3 volumes, BDF2, Jacobi PCG)",
        label="config4 ventricle shell 25/25/45 mm + 10 mm wall, P1 tets (10,276,240 nodes, "
              "59,904,000 tets), TTP06 endo/mid/epi, BDF2, dt=2e-5 s",
        window=500, cpu_steps=2),
    "cfg2": dict(
        metric="monodomain DoF*steps/s (config 2: TTP06 slab 442,401 nodes, BDF2, Jacobi PCG)",
        label="config2 TTP06 slab 20x7x3 mm h=0.1 mm (442,401 nodes), BDF2, dt=2e-5 s",
        window=250, cpu_steps=8),
}


def build_config(name):
    from paper_2308_01651_b200 import configs

    ns = configs.this_package()
    if name == "cfg4":
        from paper_2308_01651_b200 import ventricle

        return ns, ventricle.config4(ns)
    return ns, configs.config2(ns)


def probe_nodes(name, ns, cfg):
    if name == "cfg4":
        pts = [(0, 0, -45e-3), (0, 0, -55e-3), (30e-3, 0, 0), (0, 30e-3, 0),
               (-30e-3, 0, 0), (0, -30e-3, 0), (25e-3, 0, -20e-3), (0, 32e-3, -30e-3),
               (-27e-3, 0, -10e-3)]
    else:
        from paper_2308_01651_b200 import configs

        pts = configs.corner_probes() + [(10e-3, 3.5e-3, 1.5e-3)]
    return [ns.nearest_node(cfg.mesh, p) for p in pts]


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
    {"dram_bytes", "fp64_flops", "n", ...}, or None."""
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


# ---------------------------------------------------------------------------
# algorithmic bytes (DESIGN.md section 3 states the per-node
# figures): fp64, BDF2, fused design
# ---------------------------------------------------------------------------


def ionic_bytes(solver):
    """8 (3 nv + 3) per ionic DOF: read u_n, u_n-1, W_n, W_n-1; write W_n+1, c."""
    return float(sum(8 * (3 * v.num_vars + 3) * v.dofs.size for v in solver.lift_volumes))


def solve_bytes(solver, k):
    """One solve launch with k CG iterations, per node:
    RHS: combo 8 + M apply op + per lift volume (I^v 8 + op); r0 = b - A x0:
    x0 8 + op + r0 8 + D^-1 8; activation 34; reference recurrences 104 + op
    per iteration; op = bytes of one operator apply per node."""
    op = solver.op
    n = solver.n
    if op.kind == 4:                       # DIASYM: (1 + np) doubles per node
        opb = 8.0 * (1 + op.np_)
    elif op.kind == 1:                     # stencil classes: 4-byte node word
        opb = 4.0
    else:                                  # CSR / SELL: 12 B per entry
        opb = 12.0 * op.nnz / n
    nl = len(solver.lift_volumes)
    per_iter = 104.0 + opb
    fixed = 8 + opb + nl * (8 + opb) + 8 + opb + 8 + 8 + 34
    return n * (fixed + per_iter * np.asarray(k, dtype=np.float64)), opb, per_iter


def cpu_sample(name, steps, warmup=2):
    """Oracle port of the reference step (OpenMP over cells and rows, serial
    dots like the reference): `warmup` (>= 2, the BDF start-up) untimed steps
    from rest, then `steps` timed steps on the full mesh."""
    from oracle import monodomain_oracle as O

    ns, cfg = build_config(name)
    t0 = time.perf_counter()
    orc = O.OracleTissue(cfg)
    setup = time.perf_counter() - t0
    for _ in range(max(2, warmup)):
        orc.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.step()
    wall = time.perf_counter() - t0
    n = cfg.mesh.nodes.shape[0]
    return dict(value=n * steps / wall, wall=wall, cores=O.num_threads(), steps=steps,
                iters=orc.iters[max(2, warmup):], setup=setup, n=n)


def cpu_probe(kind):
    """Child process of `cpu_extras`: config 2 (442,401-node slab) on the host CPU,
    2 untimed start-up steps then 8 timed ones; prints one JSON object.
    kind "port1": the oracle port on ONE thread (OMP_NUM_THREADS=1 in the child's
    environment).  kind "numba": the UNMODIFIED reference package from baseline/_ref
    (Python + numba, all threads) through its own TissueSolver.step."""
    from paper_2308_01651_b200 import configs

    steps = 8
    if kind == "numba":
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        import numba
        from monodomain.simulation import TissueSolver as RefSolver

        cfg = configs.config2(configs.reference_namespace())
        solver = RefSolver(cfg)
        step, threads = solver.step, numba.get_num_threads()
        iters = lambda: solver.last_iterations          # noqa: E731
    else:
        from oracle import monodomain_oracle as O

        cfg = configs.config2(configs.this_package())
        solver = O.OracleTissue(cfg)
        step, threads = solver.step, O.num_threads()
        iters = lambda: solver.iters[-1]                # noqa: E731
    for _ in range(2):
        step()
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
        its.append(int(iters()))
    wall = time.perf_counter() - t0
    n = cfg.mesh.nodes.shape[0]
    print(json.dumps({"value": n * steps / wall, "unit": UNIT, "cores": threads,
                      "sample": f"config 2 ({n} nodes), {steps} steps after 2 start-up steps "
                                f"from rest (CG {min(its)}..{max(its)})"}), flush=True)


def cpu_extras():
    """Two more CPU numbers on config 2 (all cores and one thread; the
    reference's own numba path): bounded to ~a minute, failures reported in place."""
    out = {}
    for key, kind, env in (("port_one_thread_cfg2", "port1", {"OMP_NUM_THREADS": "1"}),
                           ("reference_numba_cfg2", "numba",
                            {"NUMBA_CACHE_DIR": "/tmp/numba_cache_mdx"})):
        if kind == "numba" and not (ROOT / "baseline" / "_ref" / "monodomain").is_dir():
            out[key] = {"unavailable": "baseline/_ref not installed"}
            continue
        try:
            res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cpu-probe", kind],
                                 env={**os.environ, **env}, capture_output=True, text=True,
                                 timeout=240)
            out[key] = json.loads(res.stdout.strip().splitlines()[-1])
            out[key]["kind"] = "reference" if kind == "numba" else "port"
        except Exception as exc:                       # noqa: BLE001
            out[key] = {"unavailable": f"{type(exc).__name__}: {str(exc)[:120]}"}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    steps = max(1, min(args.steps, args.ref_steps or w["cpu_steps"]))
    r = cpu_sample(args.workload, steps)
    line = {
        "impl": "reference", "metric": w["metric"], "value": r["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": 2,
        "ms_per_step": r["wall"] / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w["label"], "nodes": r["n"]},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
                         "sample": f"{steps} full step(s) after the 2 BDF start-up steps from "
                                   f"rest (CG {min(r['iters'])}..{max(r['iters'])}), full mesh, "
                                   f"oracle setup {r['setup']:.0f} s untimed"},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_window(solver, steps, dist=None, events=True):
    """K steps device-timed on the launch stream; per-step ionic/solve events."""
    import torch

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    per = []
    launches0 = solver.launches
    barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        if events:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            solver.enqueue_step(events=(e[1], e[2]))
            per.append(e)
        else:
            solver.enqueue_step()
    end.record()
    barrier()
    ms = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    its = solver.iterations_log()[-steps:]
    ionic = np.array([a.elapsed_time(b) for a, b, _ in per]) if per else None
    solve = np.array([b.elapsed_time(c) for _, b, c in per]) if per else None
    return ms, its, ionic, solve, solver.launches - launches0


def secondary_cfg2(args):
    """Config 2 from step 250 (mid-propagation), device-timed (beside the headline)."""
    from paper_2308_01651_b200.simulation import TissueSolver

    ns, cfg = build_config("cfg2")
    s = TissueSolver(cfg)
    while s.step_index < WORKLOADS["cfg2"]["window"]:
        s.enqueue_step()
    s.sync()
    ms, its, ionic, solve, _ = time_window(s, args.steps)
    b, _, _ = solve_bytes(s, its)
    step_b = b + ionic_bytes(s)
    return {"workload": WORKLOADS["cfg2"]["label"], "from_step": WORKLOADS["cfg2"]["window"],
            "value": s.n * args.steps / (ms * 1e-3), "unit": UNIT,
            "ms_per_step": ms / args.steps,
            "cg_iters_per_step": [int(its.min()), float(its.mean()), int(its.max())],
            "operator": "stencil27 class tables, SMEM-resident pipelined PCG",
            "step_frac_hbm": float(step_b.sum() / (ms * 1e-3) / 1e9 / peaks()[0])}


def run_ours(args):
    import torch

    from paper_2308_01651_b200.simulation import TissueSolver

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or os.environ.get("MDX_BENCH_DIST") == "1":
        # MDX_BENCH_DIST=1: the partitioned solver at one rank (a one-GPU pool can
        # still time its per-iteration phase path against the single-GPU kernel)
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return run_distributed(args, rank, world, local, dist)

    wl = WORKLOADS[args.workload]
    t_setup = time.perf_counter()
    ns, cfg = build_config(args.workload)
    n = cfg.mesh.nodes.shape[0]
    solver = TissueSolver(cfg)
    setup_s = time.perf_counter() - t_setup
    for _ in range(args.warmup):
        solver.enqueue_step()
    while solver.step_index < max(args.warmup, wl["window"]):
        solver.enqueue_step()
    solver.sync()
    window_from = solver.step_index
    # host copy of the window's start state (the e2e leg's input)
    # (the history levels a BDF restart of this order reads; a valid reference payload)
    payload = solver.checkpoint_payload(levels=cfg.bdf_order)

    # ---- device-timed region ------------------------------------------------
    with ClockSampler(local) as clocks:
        ms, its, ionic_ms, solve_ms, launches = time_window(solver, args.steps)

    # ---- end-to-end through the public API (host buffers) -------------------
    probes = probe_nodes(args.workload, ns, cfg)
    pidx = torch.tensor(probes, device="cuda")
    payload_pinned = torch.frombuffer(bytearray(payload), dtype=torch.uint8).pin_memory()
    del payload
    rows = torch.empty((args.steps, 2 + len(probes)), dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solver.restore(payload_pinned)
    for k in range(args.steps):
        solver.enqueue_step(record=(pidx, rows[k]))
    solver.sync()
    e2e_wall = time.perf_counter() - t0
    e2e_its = solver.iterations_log()[-args.steps:]
    assert np.isfinite(rows.numpy()).all()
    e2e = {"value": n * args.steps / e2e_wall, "unit": UNIT,
           "h2d_bytes_per_step": payload_pinned.numel() / args.steps,
           "d2h_bytes_per_step": 8 * (2 + len(probes)),
           "same_steps_as_value": bool(np.array_equal(e2e_its, its))}

    # ---- rooflines ------------------------------------------------------------
    hbm, peak_kind = peaks()
    fp64_peak, fp64_kind = fp64_peak_tflops()
    ib = ionic_bytes(solver)
    sb, opb, per_iter = solve_bytes(solver, its)
    ionic_s = float(ionic_ms.mean()) * 1e-3
    solve_share = float(solve_ms.sum() / (ionic_ms.sum() + solve_ms.sum()))
    pcg_ach = float(sb.sum() / (solve_ms.sum() * 1e-3) / 1e9)
    ion_ach = ib / ionic_s / 1e9
    step_ach = float((sb + ib).sum() / (ms * 1e-3) / 1e9)
    recur = {0: "reference CG recurrences, 3 sweeps", 1: "reference CG with q = A z + beta q, 2 sweeps",
             2: "pipelined PCG, 1 sweep"}[solver.cg_variant]
    kname = {4: f"pcg_kernel<DIASYM{solver.op.np_},tissue,NPT> ({recur})",
             3: "pcg_kernel<SELL>", 2: "pcg_kernel<CSR>",
             1: "pcg_resident_kernel<tissue>"}[solver.op.kind]
    t_pcg = traffic_of("pcg_kernel" if solver.op.kind != 1 else "pcg_resident_kernel")
    roof_pcg = {"bound": "hbm", "kernel": kname, "achieved": pcg_ach, "peak": hbm,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": pcg_ach / hbm,
                "bytes_per_launch": float(sb.mean()),
                "bytes_per_node_per_iteration": per_iter,
                "traffic": (t_pcg.get("dram_bytes") / t_pcg.get("n", n) * n
                            if t_pcg and t_pcg.get("dram_bytes") else None)}
    if roof_pcg["traffic"] and t_pcg.get("cg_iterations"):
        # the capture ran k_c CG iterations, this window's launches k on average:
        # scale the captured DRAM bytes like the algorithmic ones (once-per-launch
        # passes + per-iteration sweeps)
        fixed = float(sb.mean()) - per_iter * n * float(its.mean())
        cap = fixed + per_iter * n * t_pcg["cg_iterations"]
        roof_pcg["traffic"] *= float(sb.mean()) / cap
        roof_pcg["traffic_capture"] = {"cg_iterations": t_pcg["cg_iterations"],
                                       "dram_bytes": t_pcg["dram_bytes"]}
    t_ion = traffic_of("tissue_ionic")
    roof_ion = {"bound": "hbm", "kernel": "tissue_ionic<TTP06,2> (x3 volumes)",
                "achieved": ion_ach, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": ion_ach / hbm, "bytes_per_step": ib,
                "traffic": (t_ion.get("dram_bytes") / t_ion.get("n", n) * n
                            if t_ion and t_ion.get("dram_bytes") else None)}
    if t_ion and t_ion.get("fp64_flops"):
        flops = t_ion["fp64_flops"] / t_ion.get("n", n) * ib / 456.0
        roof_ion["fp64"] = {"achieved": flops / ionic_s / 1e12, "peak": fp64_peak,
                            "peak_kind": fp64_kind, "unit": "TFLOP/s",
                            "frac": flops / ionic_s / 1e12 / fp64_peak}
    line = {
        "metric": wl["metric"], "value": n * args.steps / (ms * 1e-3), "unit": UNIT,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["label"], "nodes": n,
                   "window": f"steps {window_from + 1}..{window_from + args.steps} "
                             f"(t = {window_from * cfg.dt * 1e3:.1f} ms on, propagation)",
                   "operator": {1: "stencil27 class tables", 2: "csr", 3: "sell32",
                                4: f"diasym ({solver.op.np_} offsets, "
                                   f"{solver.op.nrem} seam entries)"}[solver.op.kind],
                   "cg_variant": solver.cg_variant,
                   "parallelism": "single",
                   "l2": "state 3 GB and operator 0.5 GB >> 126 MB L2; no flush",
                   "cg_iters_per_step": [int(its.min()), float(its.mean()), int(its.max())],
                   "setup_s": setup_s},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
        "kernels": {"ionic_ms": float(ionic_ms.mean()), "pcg_ms": float(solve_ms.mean()),
                    "pcg_share": solve_share},
        "roofline": roof_pcg if solve_share > 0.5 else roof_ion,
        "roofline_other": roof_ion if solve_share > 0.5 else roof_pcg,
        "roofline_step": {"bound": "hbm", "achieved": step_ach, "peak": hbm, "unit": "GB/s",
                          "frac": step_ach / hbm, "bytes_per_step": float((sb + ib).mean())},
        "e2e": e2e,
    }
    del solver, payload_pinned
    torch.cuda.empty_cache()
    if args.workload == "cfg4" and not args.no_secondary:
        line["secondary"] = secondary_cfg2(args)
    if not args.no_cpu:
        r = cpu_sample(args.workload, args.cpu_steps or wl["cpu_steps"])
        line["cpu_baseline"] = {
            "value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
            "sample": f"oracle port, {r['steps']} full step(s) of the same mesh after the 2 "
                      f"BDF start-up steps from rest (CG {min(r['iters'])}..{max(r['iters'])})"}
        line["cpu_baseline"].update(cpu_extras())
    print(json.dumps(line), flush=True)


def run_distributed(args, rank, world, local, dist):
    """N > 1: the mesh partitioned over the ranks (paper_2308_01651_b200.distributed),
    strong scaling (total work fixed)."""
    import torch

    from paper_2308_01651_b200.distributed import DistributedTissueSolver

    wl = WORKLOADS[args.workload]
    ns, cfg = build_config(args.workload)
    n = cfg.mesh.nodes.shape[0]
    solver = DistributedTissueSolver(cfg)
    while solver.step_index < max(args.warmup, wl["window"]):
        solver.step()
    # the window's start state, kept in pinned host memory for the e2e leg
    snap = solver.snapshot_host()
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

    # e2e: every rank re-uploads its window-start state from pinned host
    # memory (the snapshot taken before the timed loop), runs the SAME K steps
    # through step() and reads each step's local potential range back to the host
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d = solver.restore_host(snap)
    for _ in range(args.steps):
        solver.step()
        solver.local_range().cpu()
    dist.barrier()
    torch.cuda.synchronize()
    wall = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    e2e_its = np.array(solver.iters[-args.steps:])
    if rank == 0:
        line = {
            "metric": wl["metric"], "value": n * args.steps / (ms * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["label"], "nodes": n,
                       "parallelism": solver.describe(),
                       "cg_iters_per_step": [int(its.min()), float(its.mean()),
                                             int(its.max())]},
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "e2e": {"value": n * args.steps / float(wall.item()), "unit": UNIT,
                    "h2d_bytes_per_step": h2d * world / args.steps,
                    "d2h_bytes_per_step": 16 * world,
                    "same_steps_as_value": bool(np.array_equal(e2e_its, its))},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(29500 + os.getpid() % 1000), str(ROOT / "bench.py")]
    cmd += [a for a in sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=0)
    ap.add_argument("--ref-steps", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-probe", default=None, choices=["port1", "numba"],
                    help="internal: child process of the cpu_baseline extras")
    args = ap.parse_args()
    if args.cpu_probe:
        return cpu_probe(args.cpu_probe)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
