# quick GPU check without trace: parity subset + short bench (outputs in gpurun_out/)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_precision.py -x -q -m gpu > gpurun_out/quick_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_test.log
for i in 1 2; do timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/bench_q$i.log 2>&1; done
