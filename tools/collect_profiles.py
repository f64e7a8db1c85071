"""Copy the evidence of a GPU call from gpurun_out/ into profiles/ under a round/tag prefix:
bench JSON lines, latency table, launch lists and ncu --set full summaries (dev helper).
usage: python tools/collect_profiles.py r01b"""
import csv
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio"]


def ncu_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        return "no data\n"
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = []
    for d in data:
        lines.append("---- " + d[hdr.index("Kernel Name")])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"{k:80s} {d[i]:>20s} {units[i]}")
    return "\n".join(lines) + "\n"


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    tot = {}
    for r in rows[i + 1:]:
        name = r[kn].split("(")[0]
        tot[name] = tot.get(name, 0.0) + float(r[mv].replace(",", ""))
    s = sum(tot.values())
    return "\n".join(f"{v / s:8.4f}  {v / 1e3:14.1f} us  {k}" for k, v in sorted(tot.items(), key=lambda x: -x[1]))


def main():
    tag = sys.argv[1]
    for f in sorted(glob.glob(os.path.join(OUT, "bench*.json"))):
        if os.path.getsize(f):
            shutil.copy(f, os.path.join(PROF, f"{tag}_{os.path.basename(f)}"))
    for f in ("latency.jsonl", "pytest_gpu.log", "entry_smoke.log", "smoke.log", "parity_report.jsonl", "ab.log",
              "oracle_cfg5.log"):
        p = os.path.join(OUT, f)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(PROF, f"{tag}_{f}"))
    for rep in sorted(glob.glob(os.path.join(OUT, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        with open(os.path.join(PROF, f"{tag}_{name}_ncu.txt"), "w") as fh:
            fh.write(ncu_summary(rep))
    for f in sorted(glob.glob(os.path.join(OUT, "launches*.csv"))):
        base = os.path.basename(f)[:-4]
        shutil.copy(f, os.path.join(PROF, f"{tag}_{base}.csv"))
        with open(os.path.join(PROF, f"{tag}_{base}_shares.txt"), "w") as fh:
            fh.write(launch_shares(f) + "\n")
    print("\n".join(sorted(x for x in os.listdir(PROF) if x.startswith(tag))))


if __name__ == "__main__":
    main()
