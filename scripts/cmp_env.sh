# A/B an environment knob on the C3 bench (alternating runs; prints frames/s, ms/step and the
# h_a / h_s kernel shares):  ENVS="LIC_X=1 LIC_X=0" bash scripts/cmp_env.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in ${ENVS:-base}; do
  [ "$s" = base ] && s="LIC_NONE=0"
  env $s timeout 300 python bench.py --steps ${STEPS:-150} --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_time_share']
print('$s', d['value'], d['ms_per_step'], {x: k[x] for x in k if x[0] == 'h'})"
done
