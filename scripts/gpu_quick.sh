# quick GPU check: parity subset + ga1 trace + short bench (outputs in gpurun_out/)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/quick_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_test.log
timeout 300 python scripts/trace_layer.py ${TRACE_LAYER:-ga1} > gpurun_out/trace_q.txt 2>&1
timeout 600 python bench.py --steps 100 --also "" --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_q.log
