# Round-2 final measurement pass: smoke, the bench line (both arms), the ncu
# launch list of the bench command, one ncu --set full capture of the fused
# K5q launch, per-run launch list.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r2_reference.json 2> gpurun_out/bench_r2_reference.err; echo ref_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1; echo ncub=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches.csv python tools/round_stats.py cfg5 > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:k4_round_umma -s 2 -c 1 -f -o gpurun_out/r2_k5q_fused python tools/round_stats.py cfg5 > gpurun_out/ncu_f.log 2>&1; echo ncuf=$?
