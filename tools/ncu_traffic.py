"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum per
launch) of the separable fused pipeline's six kernels from one `ncu --set full`
capture of `bench.py` at IMAGES images (six consecutive kernels of one
iteration in launch order, any starting point).  Writes the JSON bench.py reads
as roofline.traffic (profiles/r02_ncu_traffic.json: per_launch_bytes keyed by
the bench's kernel tags).  Usage: ncu_traffic.py REPORT IMAGES OUT.json"""
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
        ks.append({"kernel": r[hdr.index("Kernel Name")][:70], "bytes": rd + wr})
    assert len(ks) >= 6, "expected the six kernels of one fused iteration"
    ks = ks[:6]
    find = lambda s: next(i for i, k in enumerate(ks) if s in k["kernel"])
    ia = find("rows_t_axpy")
    cols = [i for i, k in enumerate(ks) if "cols_sep" in k["kernel"]]
    ca = (ia + 1) % 6  # the column pass right after rows_t_axpy is A's; the other is A''s
    assert ca in cols and len(cols) == 2
    cadj = next(i for i in cols if i != ca)
    tags = {"cols_sep_real#0": cadj, "rows_tt_sep#2": find("rows_tt"), "dst_tcols#2": find("dst_tcols"),
            "rows_t_axpy_sep#2": ia, "cols_sep_real#1": ca, "rows_resid_sep#1": find("resid")}
    doc = {"report": rep.split("/")[-1] + " (ncu --set full --clock-control none, bench.py C3, one iteration's six kernels)",
           "images": images, "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch",
           "per_launch_bytes": {t: ks[i]["bytes"] for t, i in tags.items()},
           "ncu_kernel_names": {t: ks[i]["kernel"] for t, i in tags.items()}}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc["per_launch_bytes"], indent=1))


if __name__ == "__main__":
    main()
