"""Summarise ncu reports (.ncu-rep) and a launch-list CSV into profiles/.

    python scripts/summarize_ncu.py <out.md> <launches.csv> <rep1> [<rep2> ...]
                                    [--n KERNEL_SUBSTRING=ROWS ...]
                                    [--iters KERNEL_SUBSTRING=K ...]

--n records how many nodes/DOFs the captured launch processed, and --iters how many
CG iterations it ran, so bench.py can scale the per-launch DRAM bytes to its own
launch size and iteration count.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def raw(rep):
    """(metrics, kernel name) of a .ncu-rep, or of its `--page raw --csv`
    export (a *_raw.csv file written on the GPU box)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")]


def fp64_flops(rep):
    """FP64 flops of the captured launch from the SASS source page
    (thread-level executed DFMA x2 + DMUL + DADD); for a *_raw.csv export the
    matching *_sass.csv next to it."""
    if rep.endswith("_raw.csv"):
        try:
            out = open(rep[:-len("_raw.csv")] + "_sass.csv").read()
        except OSError:
            return None
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3 or "Source" not in rows[1]:
        return None
    hdr = rows[1]
    i_src, i_thr = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    flops = 0
    for r in rows[2:]:
        if len(r) <= max(i_src, i_thr):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        w = {"DFMA": 2, "DMUL": 1, "DADD": 1}.get(op, 0)
        if w:
            flops += w * int(r[i_thr] or 0)
    return float(flops)


def stalls(d):
    st = []
    for k, (v, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                "_per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):
                                       -len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return sorted(st, reverse=True)[:6]


UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    import json
    from pathlib import Path

    argv = sys.argv[1:]
    sizes = {}
    while "--n" in argv:
        i = argv.index("--n")
        k, v = argv[i + 1].split("=")
        sizes[k] = int(float(v))
        del argv[i:i + 2]
    iters = {}
    while "--iters" in argv:
        i = argv.index("--iters")
        k, v = argv[i + 1].split("=")
        iters[k] = int(v)
        del argv[i:i + 2]
    out, launches, reps = argv[0], argv[1], argv[2:]
    lines = ["# ncu summary", ""]
    traffic = {}
    for rep in reps:
        d, name = raw(rep)
        try:
            tb = sum(float(d[k][0]) * UNIT[d[k][1]] for k in
                     ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            entry = {"dram_bytes": tb}
            if "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active" in d:
                entry["fp64_inst_pct_of_peak"] = float(
                    d["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"][0])
            fl = fp64_flops(rep)
            if fl:
                entry["fp64_flops"] = fl
            for k, v in sizes.items():
                if k in name:
                    entry["n"] = v
            for k, v in iters.items():
                if k in name:
                    entry["cg_iterations"] = v
            traffic[name.split("(")[0]] = entry
        except (KeyError, ValueError):
            pass
        lines += [f"## `{name[:110]}`", "", f"report: `{rep}`", "",
                  "| metric | value | unit |", "|---|---|---|"]
        for key, label in METRICS:
            if key in d:
                v, u = d[key]
                lines.append(f"| {label} (`{key}`) | {v} | {u} |")
        lines += ["", "top stall reasons (warps per issued instruction): " +
                  ", ".join(f"{n} {v:.2f}" for v, n in stalls(d)), ""]
    # launch list: share of device time per kernel
    rows = ([] if launches == "-" else
            list(csv.DictReader(l for l in open(launches) if not l.startswith("=="))))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1.0)
        tot[k] += v * scale
        cnt[k] += 1
    all_t = sum(tot.values()) or 1.0
    lines += ["## launch list (ncu, --clock-control none, serialised, cold cache)", "",
              "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k[:80]}` | {cnt[k]} | {v:.1f} | {v / all_t:.1%} |")
    open(out, "w").write("\n".join(lines) + "\n")
    (Path(out).parent / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
