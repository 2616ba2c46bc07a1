python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for l in ga4 ha1 ha2 ha3 hs1 hs2 hs3 gs1 gs4; do echo "== $l"; timeout 300 python scripts/trace_layer.py $l 2>&1 | tail -3; done > gpurun_out/trace_all.txt
