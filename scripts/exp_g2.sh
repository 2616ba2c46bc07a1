python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
LIC_G2=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_precision.py -x -q -m gpu > gpurun_out/g2_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g2_test.log
for v in 1 2; do LIC_G2=$v timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/bench_g2_$v.log 2>&1; done
LIC_G2=2 TRACE_LAYER=gs3 timeout 300 python scripts/trace_layer.py gs3 > gpurun_out/trace_gs3_g2.txt 2>&1
