# bench.py under several environment settings (VARIANTS: ';'-separated env assignment lists), 2 rounds
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
IFS=';' read -ra V <<< "$VARIANTS"
for r in 1 2; do
  i=0
  for v in "${V[@]}"; do
    env $v timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/mv_${i}_$r.log 2>&1
    echo "$i: $v" > gpurun_out/mv_${i}.name
    i=$((i+1))
  done
done
