python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python scripts/trace_layer.py hs3 > gpurun_out/trace_hs3b.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sigma or index or encode_planes" > gpurun_out/t_hs3.log 2>&1; echo rc=$? >> gpurun_out/t_hs3.log
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg --clock-control none -k regex:conv_umma -s 17 -c 17 --csv --log-file gpurun_out/step_metrics2.csv python scripts/profile_step.py > gpurun_out/ncu_step.log 2>&1
