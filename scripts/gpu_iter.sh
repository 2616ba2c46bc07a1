# one build -> measure iteration on the GPU box: gpu tests, per-tile traces, bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for L in ${TRACE_LAYERS:-ga1 gs3}; do echo "== trace $L"; timeout 120 python scripts/trace_layer.py $L 2>&1 | tail -2; done
timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['latency_ms']['p50'], d['busy'], d['roofline']['frac']); print(d['kernel_time_share'])"
