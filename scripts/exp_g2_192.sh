python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -m gpu -s > gpurun_out/g192_test.log 2>&1; echo "rc=$?" >> gpurun_out/g192_test.log
cat > /tmp/plan4.py <<'PY'
import sys; sys.path.insert(0, '.')
from lic_synth import ModelSpec, generate_weights, write_licw
from paper_2208_01641_b200 import lic
spec = ModelSpec(kind=1, N=192, M=320)
c = lic.Codec(write_licw(spec, generate_weights(spec, 0)), 720, 1280, max_batch=4)
PY
LIC_PLAN_DEBUG=1 python /tmp/plan4.py > gpurun_out/plan_c4.txt 2>&1
for i in 1 2; do
  LIC_G2_192=0 timeout 600 python bench.py --config c4 --steps 60 --also "" --no-cpu-baseline > gpurun_out/c4_A$i.log 2>&1
  timeout 600 python bench.py --config c4 --steps 60 --also "" --no-cpu-baseline > gpurun_out/c4_B$i.log 2>&1
done
