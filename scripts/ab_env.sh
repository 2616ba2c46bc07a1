# A/B: bench.py under two environment settings, interleaved ($A, $B: env assignments, e.g. "LIC_G2=1")
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do
  env $A timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_A$i.log 2>&1
  env $B timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_B$i.log 2>&1
done
