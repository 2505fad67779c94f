"""Summarises an ncu --set full report and a launch-list CSV into markdown
(run here, on the CPU box, on files brought back in gpurun_out/)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%active"),
    ("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_thru_%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefront_%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
]
# warp stall reasons, cycles per issued instruction
STALLS = ["wait", "short_scoreboard", "barrier", "no_instruction", "long_scoreboard", "not_selected",
          "math_pipe_throttle", "mio_throttle", "branch_resolving", "dispatch_stall"]


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(k[1] for k in KEYS) + " |", "|---" * (len(KEYS) + 1) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "")[:48]
        vals = []
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        out.append(f"| {name} | " + " | ".join(vals) + " |")
    out += ["", "Warp stalls per issued instruction (smsp__average_warps_issue_stalled_*_per_issue_active):", "",
            "| kernel | " + " | ".join(STALLS) + " |", "|---" * (len(STALLS) + 1) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "")[:48]
        vals = []
        for st in STALLS:
            k = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
            vals.append(r[hdr.index(k)] if k in hdr else "-")
        out.append(f"| {name} | " + " | ".join(vals) + " |")
    return "\n".join(out)


def launch_list(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        tot[k] += float(r["Metric Value"])
        cnt[k] += 1
    s = sum(tot.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {100 * v / s:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(full_report(path) if mode == "full" else launch_list(path))
