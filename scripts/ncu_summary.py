"""Summarise an ncu --set full capture of scripts/profile_step.py into profiles/.

    python scripts/ncu_summary.py gpurun_out/full.ncu-rep profiles/r1_ncu_full_summary_vN.csv "header note"

Kernel order of profile_step.py (17 conv_umma launches per pass):
ga1 ga2 ga3 ga4 ha1 ha2 ha3 hs1 hs2 hs3 | hs1 hs2 hs3 (decoder GPU1) | gs1 gs2 gs3 gs4.
Also rewrites profiles/ncu_traffic.json (dram read + write bytes per launch) which
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

NAMES = ["ga1", "ga2", "ga3", "ga4", "ha1", "ha2", "ha3", "hs1", "hs2", "hs3",
         "hs1_dec", "hs2_dec", "hs3_dec", "gs1", "gs2", "gs3", "gs4"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread"]


def main(rep, out, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {m: hdr.index(m) for m in METRICS}
    lines = [f"# {note}",
             "# scripts/profile_step.py (batch 4 frames, 1280x720 hyper 128/192); one launch per kernel; "
             "cold-cache serialised replays",
             "# units: " + ", ".join(f"{m}[{units[col[m]]}]" for m in METRICS),
             "kernel," + ",".join(METRICS)]
    traffic = {}
    for name, r in zip(NAMES, data):
        lines.append(name + "," + ",".join(r[col[m]] for m in METRICS))
        mb = float(r[col["dram__bytes_read.sum"]]) + float(r[col["dram__bytes_write.sum"]])
        unit = units[col["dram__bytes_read.sum"]]
        scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}[unit]
        if not name.endswith("_dec"):
            traffic[name] = mb * scale
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    traffic["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (batch 4), ncu --set full, "
                        f"{os.path.basename(out)}")
    tpath = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
