# env sweep on one bench config: SWEEP="NAME=VAL;NAME=VAL ..." (space-separated settings), CONFIG=c3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for s in ${SWEEP:-base}; do
  envs=$(echo "$s" | tr ';' ' ')
  [ "$s" = base ] && envs=""
  env $envs LIC_PLAN_DEBUG=1 timeout 300 python bench.py --config ${CONFIG:-c3} --steps ${STEPS:-100} --no-cpu-baseline > gpurun_out/sweep.log 2>gpurun_out/sweep.err
  echo "== $s rc=$?"
  [ -n "$PLAN" ] && sort -u gpurun_out/sweep.err | grep "^plan" | head -20
  tail -1 gpurun_out/sweep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac']); print({k:v for k,v in list(d['kernel_time_share'].items())[:6]})" 2>&1 | tail -2
done
