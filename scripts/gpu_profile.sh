# ncu evidence for profiles/: launch list of a short bench run + one --set full capture of every
# GEMM-engine launch of one encode + hyper_indexes + decode pass (scripts/profile_step.py)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_umma -s 17 -c 17 -o gpurun_out/full python scripts/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
