# Round-2 (third session, final code: + hi-only g_s L1 plan, 3000-frame default bench run) evidence for profiles/ (run on the GPU box from the repo root; outputs in gpurun_out/):
# launch list of a short bench run, one ncu --set full capture of every GEMM-engine launch of
# one encode + hyper_indexes + decode pass, the default bench line, the other configs, the
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2f_smoke.log
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 4 --warmup 3 --also "" --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_umma -s 17 -c 17 -o gpurun_out/r2f_full python scripts/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
NO_BUILD=1 NCU_OUT=r2f_step_metrics bash scripts/gpu_ncu_step.sh
timeout 900 python bench.py --timeline-out gpurun_out/r2f_timeline_c3.json > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
for cfg in c2 c4 c5; do timeout 600 python bench.py --config $cfg --also "" --no-cpu-baseline --steps 100 >> gpurun_out/r2f_bench_configs.jsonl 2>> gpurun_out/r2f_bench.err; done
for v in "--precision f16" "--activation 1dn" "--coder rans64" "--zero-copy" "--batch 8"; do echo "# $v" >> gpurun_out/r2f_bench_variants.jsonl; timeout 600 python bench.py $v --also "" --no-cpu-baseline --steps 100 >> gpurun_out/r2f_bench_variants.jsonl 2>> gpurun_out/r2f_bench.err; done
echo "# LIC_L1_ROWS=0 (im2col g_a L1 tiles)" >> gpurun_out/r2f_bench_variants.jsonl; LIC_L1_ROWS=0 timeout 600 python bench.py --also "" --no-cpu-baseline --steps 100 >> gpurun_out/r2f_bench_variants.jsonl 2>> gpurun_out/r2f_bench.err
echo done
