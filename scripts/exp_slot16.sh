python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu -s > gpurun_out/s16_test.log 2>&1; echo "rc=$?" >> gpurun_out/s16_test.log
LIC_G2_SLOT16=0 NO_BUILD=1 NCU_OUT=s16_0 bash scripts/gpu_ncu_step.sh
NO_BUILD=1 NCU_OUT=s16_1 bash scripts/gpu_ncu_step.sh
for i in 1 2; do
  LIC_G2_SLOT16=0 timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/s16_A$i.log 2>&1
  timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/s16_B$i.log 2>&1
  LIC_G2_SLOT16=0 timeout 600 python bench.py --config c4 --steps 60 --also "" --no-cpu-baseline > gpurun_out/s16_C4A$i.log 2>&1
  timeout 600 python bench.py --config c4 --steps 60 --also "" --no-cpu-baseline > gpurun_out/s16_C4B$i.log 2>&1
done
