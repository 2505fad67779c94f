"""Per-class DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
the fused pipeline's kernels from one `ncu --set full` capture of
`bench.py --images IMAGES` (six consecutive kernels of one iteration in launch order, any
starting point: conv_col(A'), rows_ainv_tt, dst_tcols, rows_t_axpy_afwd,
conv_col(A), rows_ainv_resid).  Writes the per-image, per-launch bytes bench.py reports as
roofline.traffic.  Usage: ncu_traffic.py REPORT IMAGES OUT.json"""
import csv
import io
import json
import subprocess
import sys

def main():
    rep, images, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ks = []
    for r in rows[2:]:
        rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
        ks.append({"kernel": r[hdr.index("Kernel Name")][:60], "bytes": rd + wr})
    assert len(ks) >= 6, "expected the six kernels of one fused iteration"
    ks = ks[:6]
    # the column pass right after rows_t_axpy is A's (blur class); the other is A'
    is_col = lambda k: "conv_col" in k["kernel"] or "cols_sep" in k["kernel"]
    ia = next(i for i, k in enumerate(ks) if "rows_t_axpy" in k["kernel"])
    conv = [i for i, k in enumerate(ks) if is_col(k)]
    ca = (ia + 1) % 6 if (ia + 1) % 6 in conv else conv[0]
    cadj = next(i for i in conv if i != ca)
    find = lambda s: next(i for i, k in enumerate(ks) if s in k["kernel"])
    resid = next(i for i, k in enumerate(ks) if "resid" in k["kernel"])
    classes = {"blur_adjoint(A')": [cadj],
               "ar_transform_pass": [find("rows_ainv_tt"), find("dst_tcols"), ia],
               "blur(A)+residual": [ca, resid]}
    per = {c: sum(ks[i]["bytes"] for i in idx) / len(idx) / images for c, idx in classes.items()}
    json.dump({"report": rep.split("/")[-1], "images": images, "kernels": ks[:6],
               "per_image_launch_bytes": per}, open(out, "w"), indent=1)
    print(json.dumps(per, indent=1))


if __name__ == "__main__":
    main()
