# ga1 / hyper-layer evidence: per-tile timelines and one ncu --set full capture with source
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for l in ga1 gs3 ha3 hs3; do timeout 300 python scripts/trace_layer.py $l > gpurun_out/trace_$l.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_umma -s 17 -c 1 -o gpurun_out/ga1_full python scripts/profile_step.py > gpurun_out/ncu_ga1.log 2>&1; echo "ncu ga1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_umma -s 23 -c 1 -o gpurun_out/ha3_full python scripts/profile_step.py > gpurun_out/ncu_ha3.log 2>&1; echo "ncu ha3 rc=$?"
echo done
