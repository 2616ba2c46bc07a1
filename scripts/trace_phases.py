"""Mean per-tile epilogue phase times (cycles after the epilogue start) of a trace_layer.py dump.

    python scripts/trace_phases.py gpurun_out/trace_ga1.txt
"""
import sys

lines = open(sys.argv[1]).read().splitlines()
h0 = next(i for i, l in enumerate(lines) if l.split()[:1] == ["tile"])      # (skips plan-debug lines)
hdr = lines[h0].split()
rows = [l.split() for l in lines[h0 + 1:] if l.strip() and l.split()[0].isdigit()]
ix = {h: i for i, h in enumerate(hdr)}
rows = rows[4:-2] if len(rows) > 8 else rows
acc = {}
for r in rows:
    e = int(r[ix["epi_s"]])
    for k in ("epi_x2", "epi_n", "epi_p2", "epi_stg", "epi_acq", "epi_e"):
        v = int(r[ix[k]])
        if v >= 0:
            acc.setdefault(k, []).append(v - e)
per = [int(rows[i + 1][ix["mma_s"]]) - int(rows[i][ix["mma_s"]]) for i in range(len(rows) - 1)]
print(" ".join(f"{k} {sum(v) / len(v):.0f}" for k, v in acc.items()), f"| period {sum(per) / max(1, len(per)):.0f}")
