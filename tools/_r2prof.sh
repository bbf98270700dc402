# Round-2 measurement pass: tests, smoke, the bench line, the launch list of
# full config-5 runs, and one ncu --set full capture of the fused K5q launch.
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches.csv python tools/round_stats.py cfg5 > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:k4_round_umma -s 2 -c 1 -f -o gpurun_out/r2_k5q_fused python tools/round_stats.py cfg5 > gpurun_out/ncu_f.log 2>&1; echo ncuf=$?
