cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/t_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python tools/round_stats.py cfg5 > gpurun_out/round_stats.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:k4_round_umma -c 1 -o gpurun_out/k5q_w3 -f python tools/profile_round.py cfg5 8 --upper=18 > gpurun_out/ncu_k5q.log 2>&1; echo ncuf=$?
