#!/usr/bin/env python
"""Copy a measurement round's evidence from gpurun_out/ (scratch) into profiles/
(tracked): bench lines, the launch lists, ncu summaries of the full captures (raw
metrics of interest + per-source-line tables), sanitizer / test / smoke logs.

    python scripts/collect_profiles.py r02
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = "gpurun_out", "profiles"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
           "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]


def bench_lines(path):
    out = []
    for line in open(path, errors="replace"):
        if line.startswith("{"):
            out.append(json.loads(line))
    return out


def main():
    os.makedirs(P, exist_ok=True)
    b = bench_lines(f"{G}/{TAG}_bench.log")
    if b:
        json.dump(b[-1], open(f"{P}/{TAG}_bench.json", "w"), indent=1)
    r = bench_lines(f"{G}/{TAG}_reference.log")
    if r:
        json.dump(r[-1], open(f"{P}/{TAG}_reference.json", "w"), indent=1)
    with open(f"{P}/{TAG}_configs.jsonl", "w") as f:
        for c in ("C1", "C2", "C4", "C5", "C6"):
            p = f"{G}/{TAG}_bench_{c}.log"
            if os.path.exists(p):
                for d in bench_lines(p):
                    f.write(json.dumps(d) + "\n")
    for name in (f"{TAG}_launches.csv", f"{TAG}_launches_C2.csv", f"{TAG}_launches_C4.csv"):
        if os.path.exists(f"{G}/{name}"):
            shutil.copy(f"{G}/{name}", f"{P}/{name}")
    for name in ("tests.log", "smoke.log", "sanitize_memcheck.log", "sanitize_racecheck.log",
                 "sanitize_synccheck.log", "sanitize_initcheck.log"):
        src = f"{G}/{TAG}_{name}"
        if os.path.exists(src) and "closed on this pool" not in open(src, errors="replace").read():
            shutil.copy(src, f"{P}/{TAG}_{name}")
    summary = {}
    for cfg in ("C3", "C2"):
        rep = f"{G}/{TAG}_full_{cfg}.ncu-rep"
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        for i, row in enumerate(rows[2:]):
            k = row[h.index("Kernel Name")]
            summary[f"{cfg}#{i} {k[:90]}"] = {m: f"{row[h.index(m)]} {units[h.index(m)]}".strip()
                                            for m in METRICS if m in h}
        for kre in (["hot_compose", "bucket_coarse", "part_scatter"] if cfg == "C3" else ["bucket_warp", "part_scatter"]):
            txt = subprocess.run([sys.executable, "scripts/ncu_lines.py", rep, kre, "0", "30"],
                                 capture_output=True, text=True).stdout
            open(f"{P}/{TAG}_ncu_lines_{cfg}_{kre}.txt", "w").write(txt)
    if summary:
        json.dump(summary, open(f"{P}/{TAG}_ncu_full_summary.json", "w"), indent=1)
    print("collected", TAG)


if __name__ == "__main__":
    main()
