"""Per-CUDA-source-line stall samples and executed instructions of one kernel launch in an
ncu report (--import-source on, -lineinfo).

    python scripts/ncu_lines.py gpurun_out/full.ncu-rep <launch index> [top]
"""
import csv
import io
import os
import subprocess
import sys


def main(rep, idx, top=40):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:conv", "--launch-skip", str(idx), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    fname, hdr, recs = "?", None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1]); continue
        if r[0] == "Line No":
            hdr = r; continue
        if hdr is None or len(r) < len(hdr) - 5 or not r[0].isdigit() or r[2] != "-":
            continue
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            ex = int(r[hdr.index("Instructions Executed")])
        except ValueError:
            continue
        recs.append((s, ex, fname, int(r[0]), r[1]))
    tot_s = sum(x[0] for x in recs); tot_e = sum(x[1] for x in recs)
    print(f"total samples {tot_s} instr {tot_e}")
    for s, ex, f, ln, src in sorted(recs, reverse=True)[:int(top)]:
        print(f"{f[:10]:10s}:{ln:<5d} {s:7d} {100*s/max(1,tot_s):5.1f}%  instr {100*ex/max(1,tot_e):5.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
