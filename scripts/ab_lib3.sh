# A/B of two in-tree builds (liblic_a.so = A, liblic.so = B): 3 interleaved bench pairs + ncu step metrics
for i in 1 2 3; do
  LIC_LIB=liblic_a.so timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_A$i.log 2>&1
  timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_B$i.log 2>&1
done
LIC_LIB=liblic_a.so NO_BUILD=1 NCU_OUT=ab_stepA bash scripts/gpu_ncu_step.sh
NO_BUILD=1 NCU_OUT=ab_stepB bash scripts/gpu_ncu_step.sh
