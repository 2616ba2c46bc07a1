# one ncu --set full capture (with source) of launch $NCU_S of scripts/profile_step.py + a trace of $TRACE_LAYER
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/trace_layer.py ${TRACE_LAYER:-ga1} > gpurun_out/trace_q.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_umma -s ${NCU_S:-17} -c 1 -o gpurun_out/${NCU_NAME:-k_full} python scripts/profile_step.py > gpurun_out/ncu_k.log 2>&1; echo "ncu rc=$?"
