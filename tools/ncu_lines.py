"""Per-source-line warp-stall samples of one kernel from an ncu report
(`--page source --print-source cuda,sass`), top lines first.  Diagnostic.
Usage: ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    fname, lines, tot = "?", [], 0.0
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif len(r) > 4 and r[0].isdigit() and r[2] == "-":
            try:
                v = float(r[4])
            except ValueError:
                continue
            lines.append((v, fname, int(r[0]), r[1].strip()))
            tot += v
    lines.sort(reverse=True)
    print(f"total stall samples {tot:.0f}")
    for v, f, n, src in lines[:top]:
        print(f"{100 * v / tot:5.1f}%  {f}:{n}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
