python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py tests/test_gpu_chained_fullsize.py tests/test_gpu_pipeline.py -x -q -m gpu > gpurun_out/ks_test.log 2>&1; echo "rc=$?" >> gpurun_out/ks_test.log
timeout 300 python scripts/dbg/determinism.py 20 > gpurun_out/ks_det.log 2>&1
NO_BUILD=1 NCU_OUT=ks_step1 bash scripts/gpu_ncu_step.sh
LIC_KSPLIT=0 NO_BUILD=1 NCU_OUT=ks_step0 bash scripts/gpu_ncu_step.sh
for i in 1 2; do
  LIC_KSPLIT=0 timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_A$i.log 2>&1
  timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/ab_B$i.log 2>&1
done
