python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q -m gpu -s > gpurun_out/var_test.log 2>&1; echo "rc=$?" >> gpurun_out/var_test.log
timeout 300 python scripts/dbg/determinism.py 30 > gpurun_out/determinism.log 2>&1
LIC_SMALL_BN=64 timeout 300 python scripts/dbg/determinism.py 30 > gpurun_out/determinism_sbn.log 2>&1
NCU_OUT=step_mn1 bash scripts/gpu_ncu_step.sh; LIC_G2_MMANORM=0 NCU_OUT=step_mn0 bash scripts/gpu_ncu_step.sh
