"""Per-kernel LSU / shared-memory pressure of an ncu --set full report with
sources: pipe utilisations, bank conflicts, and the source lines with the most
excess shared-memory wavefronts.  Diagnostic.  Usage: ncu_excess.py REPORT [TOP]"""
import csv
import io
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "time"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
        ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "lsu_wavefronts_%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefronts_%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
        ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%")]


def main(rep, top=8):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    seen = set()
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if name in seen:
            continue
        seen.add(name)
        print("##", name[:90])
        print("  " + ", ".join(f"{lab}={r[h.index(k)]}" for k, lab in WANT if k in h))
        stalls = sorted(((float(r[i]), k.split("issue_stalled_")[1].split("_per_issue")[0]) for i, k in enumerate(h)
                         if "issue_stalled" in k and k.endswith("per_issue_active.ratio") and r[i] not in ("", "n/a")),
                        reverse=True)[:6]
        print("  stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls))
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                              "--launch-skip",
                              r[h.index("ID")], "--launch-count", "1"], capture_output=True, text=True).stdout
        hdr, cur, lines = None, "?", []
        for q in csv.reader(io.StringIO(src)):
            if not q:
                continue
            if q[0] == "File Path":
                cur = q[1].split("/")[-1]
            elif q[0] == "Line No":
                hdr = q
            elif hdr and q[0].isdigit() and len(q) == len(hdr):
                d = dict(zip(hdr, q))
                try:
                    lines.append((float(d["L1 Wavefronts Shared Excessive"] or 0), float(d["L1 Wavefronts Shared"] or 0),
                                  cur, q[0], q[1].strip()[:80]))
                except (KeyError, ValueError):
                    pass
        tot = sum(x[1] for x in lines) or 1.0
        for ex, wf, f, ln, s in sorted(lines, reverse=True)[:top]:
            if ex > 0:
                print(f"  excess {100 * ex / tot:5.1f}% of smem wavefronts ({wf / tot * 100:4.1f}% total)  {f}:{ln}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
