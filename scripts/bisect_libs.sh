# ncu step metrics for several in-tree library builds (LIBS: space-separated liblic_*.so names)
for L in $LIBS; do
  LIC_LIB=$L NO_BUILD=1 NCU_OUT=bis_$L bash scripts/gpu_ncu_step.sh
done
for L in $LIBS; do
  LIC_LIB=$L timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/bis_$L.log 2>&1
done
