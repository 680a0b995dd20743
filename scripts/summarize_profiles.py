"""Distill ncu captures and launch lists (gpurun_out/) into profiles/<tag>_*.

  python scripts/summarize_profiles.py r01 [RUN]

RUN selects one gpu_iter.sh run (gpurun_out/{prof,launches,bench}_RUN.*);
without it every .ncu-rep in gpurun_out/ is summarised.

Writes profiles/<tag>_ncu_summary.md (key metrics + top stall reasons + the
hottest source lines per kernel), profiles/<tag>_launches.csv (per-launch
device times of the bench-shaped run) and copies the bench line.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "CTA limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
]


def ncu_csv(args):
    r = subprocess.run(["ncu", *args], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def _bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def _num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def summarize(rep, fh, traffic, kernels=None):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    if len(rows) < 3:
        return
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if kernels is not None:  # machine-readable per-kernel figures (bench.py roofline.kernels)
            def get(key, scale=1.0):
                return _num(r[h.index(key)]) * scale if key in h and _num(r[h.index(key)]) is not None else None
            it = h.index("gpu__time_duration.sum") if "gpu__time_duration.sum" in h else None
            dur_scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(units[it], 1.0) if it is not None else 1.0
            rec = {"capture": os.path.basename(rep),
                   "duration_ms": get("gpu__time_duration.sum", dur_scale),
                   "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "fp64_pipe_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                   "alu_pipe_pct": get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                   "fma_pipe_pct": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                   "warps_active_per_sm": get("sm__warps_active.avg.per_cycle_active"),
                   "registers": get("launch__registers_per_thread"),
                   "warp_instructions": get("smsp__inst_executed.sum"),
                   "l1_wavefronts_pct": get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")}
            if "dram__bytes_read.sum" in h and "dram__bytes_write.sum" in h:
                ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
                rec["dram_bytes"] = _bytes(r[ir], units[ir]) + _bytes(r[iw], units[iw])
            if "lts__t_bytes.sum" in h:
                il = h.index("lts__t_bytes.sum")
                rec["l2_bytes"] = _bytes(r[il], units[il])
            kernels.setdefault(name.split("(")[0], []).append(rec)
        if "dram__bytes_read.sum" in h and "dram__bytes_write.sum" in h:
            ir, iw, it = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
            traffic.setdefault(name.split("(")[0], []).append(
                {"dram_bytes": _bytes(r[ir], units[ir]) + _bytes(r[iw], units[iw]),
                 "dram_read_bytes": _bytes(r[ir], units[ir]), "dram_write_bytes": _bytes(r[iw], units[iw]),
                 "duration": r[it] + " " + units[it], "capture": os.path.basename(rep)})
        fh.write(f"\n### `{name}`\n\n| metric | value |\n|---|---|\n")
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                fh.write(f"| {label} | {r[i]} {units[i]} |\n")
        st = [(h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(r[i])) for i in range(len(h))
              if "average_warps_issue_stalled" in h[i] and "per_issue_active" in h[i] and r[i] not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        fh.write("\nTop stall reasons (warps per issued instruction): "
                 + ", ".join(f"{a} {b:.2f}" for a, b in st[:6]) + "\n")
        kname = name.split("(")[0].split("<")[0].split()[-1].split("::")[-1]
        src = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", f"regex:{kname}"])
        hi = [i for i, x in enumerate(src) if x and x[0] == "Line No"]
        if not hi:
            continue
        hdr = src[hi[0]]
        idx = {x: i for i, x in enumerate(hdr)}
        recs = []
        for x in src[hi[0] + 1:]:
            if len(x) < len(hdr) or x[2] != "-":
                continue
            try:
                recs.append((int(x[0]), x[1].strip()[:80], int(x[idx["# Samples"]] or 0),
                             int(x[idx["Instructions Executed"]] or 0)))
            except ValueError:
                pass
        ts = sum(x[2] for x in recs) or 1
        ti = sum(x[3] for x in recs) or 1
        fh.write("\nHottest source lines (share of stall samples / of instructions):\n\n")
        for x in sorted(recs, key=lambda x: -x[2])[:8]:
            fh.write(f"- line {x[0]}: {100 * x[2] / ts:.1f}% samples, {100 * x[3] / ti:.1f}% instr — `{x[1]}`\n")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    run = sys.argv[2] if len(sys.argv) > 2 else None
    os.makedirs(PROF, exist_ok=True)
    reps = ([f for f in (f"prof_{run}.ncu-rep", f"prof_train_{run}.ncu-rep") if os.path.exists(os.path.join(OUT, f))]
            if run else sorted(f for f in os.listdir(OUT) if f.endswith(".ncu-rep")))
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write(f"# ncu summary ({tag})\n\nFrom `ncu --set full --clock-control none --import-source on` "
                 "captures (cold-cache, serialised replays: compare shares, not absolutes).\n")
        traffic, kernels = {}, {}
        for rep in reps:
            fh.write(f"\n## {rep}\n")
            summarize(os.path.join(OUT, rep), fh, traffic, kernels)
    with open(os.path.join(PROF, f"{tag}_kernels.json"), "w") as g:
        json.dump(kernels, g, indent=1)
    # per-launch DRAM traffic of each captured kernel (bench.py roofline.traffic)
    with open(os.path.join(PROF, f"{tag}_traffic.json"), "w") as g:
        json.dump(traffic, g, indent=1)
    if run:
        for src, dst in ((f"launches_{run}.csv", "launches.csv"), (f"launches_train_{run}.csv", "launches_train.csv"),
                         (f"bench_{run}.json", "bench.json")):
            if os.path.exists(os.path.join(OUT, src)):
                import shutil
                shutil.copy(os.path.join(OUT, src), os.path.join(OUT, dst))
    for f in ("launches.csv", "launches_train.csv"):
        src = os.path.join(OUT, f)
        if os.path.exists(src):
            rows = [r for r in csv.reader(open(src)) if len(r) > 10]
            with open(os.path.join(PROF, f"{tag}_{f}"), "w", newline="") as g:
                w = csv.writer(g)
                w.writerow(["kernel", "gpu__time_duration.sum (ns)"])
                for r in rows[1:]:
                    if "snn" in r[4] or "k_" in r[4]:
                        w.writerow([r[4], r[-1]])
    b = os.path.join(OUT, "bench.json")
    if os.path.exists(b):
        line = open(b).read().strip().splitlines()[-1]
        json.loads(line)
        with open(os.path.join(PROF, f"{tag}_bench.json"), "w") as g:
            g.write(line + "\n")


if __name__ == "__main__":
    main()
