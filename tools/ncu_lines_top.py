"""Top source lines of an ncu --page source --csv --print-source cuda,sass export
by warp-stall samples (with smem conflicts): python tools/ncu_lines_top.py FILE [N]"""
import csv
import sys

rows, cur = [], None
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "":
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        conf = d.get("L1 Conflicts Shared N-Way", "0")
        ex = d.get("L1 Wavefronts Shared Excessive", "0")
        rows.append((s, cur, r[0], r[1].strip()[:90], ex))
tot = sum(x[0] for x in rows)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total samples {tot}")
for s, f, ln, src, ex in sorted(rows, reverse=True)[:N]:
    print(f"{100*s/tot:5.1f}% {f}:{ln} smem_excess={ex}  {src}")
