# A/B of two in-tree builds: liblic_a.so (A) vs liblic.so (B), ncu step metrics + interleaved benches
timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/ab_test.log 2>&1; echo "rc=$?" >> gpurun_out/ab_test.log
LIC_LIB=liblic_a.so NO_BUILD=1 NCU_OUT=ab_stepA bash scripts/gpu_ncu_step.sh
NO_BUILD=1 NCU_OUT=ab_stepB bash scripts/gpu_ncu_step.sh
for i in 1 2; do
  LIC_LIB=liblic_a.so timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_A$i.log 2>&1
  timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_B$i.log 2>&1
done
