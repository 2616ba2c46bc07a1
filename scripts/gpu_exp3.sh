mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for L in gs3 ga1; do
for cfg in "LIC_DBG_NOSTORE=0" "LIC_DBG_NOSTORE=1" "LIC_DBG_NOSTORE=8" "LIC_DBG_NOSTORE=16" "LIC_DBG_NOSTORE=24"; do
  echo "== $L $cfg"; env $cfg timeout 120 python scripts/trace_layer.py $L > /tmp/t.txt 2>&1; tail -2 /tmp/t.txt; sed -n 8,9p /tmp/t.txt | cut -c1-120
done; done
