"""Table of the per-kernel metrics written by scripts/gpu_ncu_step.sh (ncu --csv log)."""
import collections, csv, sys
f = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/step_metrics.csv"
lines = [l for l in open(f) if not l.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]
iid, im, iv = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
names = "ga1 ga2 ga3 ga4 ha1 ha2 ha3 hs1 hs2 hs3 hs1d hs2d hs3d gs1 gs2 gs3 gs4".split()
d = collections.defaultdict(dict)
for r in rows[1:]:
    if len(r) > iv:
        d[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
ids = sorted(d)
tot = sum(d[i]["gpu__time_duration.sum"] for i in ids)
for n, i in zip(names, ids):
    m = d[i]
    print(f"{n:5s} {m['gpu__time_duration.sum'] / 1000:8.1f} us ({100 * m['gpu__time_duration.sum'] / tot:4.1f}%)  tensor "
          f"{m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']:5.1f}%  issue "
          f"{m['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f}%  dram "
          f"{(m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']) / 1e6:7.1f} MB")
print(f"total {tot / 1000:.1f} us")
