# A/B of environment switches on one box: bench.py per setting, interleaved twice
# usage: AB="LIC_X=0|LIC_X=1" bash scripts/ab_bench.sh  (outputs gpurun_out/ab_*.json, summary on stdout)
mkdir -p gpurun_out
[ -n "$NO_BUILD" ] || python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
IFS='|' read -ra SETS <<< "$AB"
for rep in 1 2; do
  for i in "${!SETS[@]}"; do
    env ${SETS[$i]} timeout 300 python bench.py --no-cpu-baseline --also "" ${BENCH_ARGS} > gpurun_out/ab_${i}_${rep}.json 2>/dev/null
    python - "$i" "$rep" "${SETS[$i]}" <<'PY'
import json, sys
i, rep, s = sys.argv[1:]
try:
    d = json.load(open(f"gpurun_out/ab_{i}_{rep}.json"))
    L = d["layers"]
    print(f"{s:28s} rep{rep} fps {d['value']:8.1f} e2e {d['e2e']['value']:8.1f} mhz {d['clocks']['sm_mhz']:6.0f} " +
          " ".join(f"{k} {L[k]['ms_per_launch']*1000:.0f}" for k in ("ga1", "ga2", "ga3", "gs1", "gs2", "gs3", "gs4") if k in L))
except Exception as e:
    print(s, rep, "failed", e)
PY
  done
done
