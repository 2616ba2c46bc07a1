# per-kernel summary metrics of one profiled pass of scripts/profile_step.py (launches 17..33)
mkdir -p gpurun_out
[ -n "$NO_BUILD" ] || python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg --clock-control none -k regex:conv_umma -s 17 -c 17 --csv --log-file gpurun_out/${NCU_OUT:-step_metrics}.csv python scripts/profile_step.py > gpurun_out/ncu_step.log 2>&1; echo "ncu rc=$?"
