cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 16 3 5 6 17 21 23; do
  for r in 1 2; do echo "debug=$d"; BZ_K4_DEBUG=$d python tools/profile_round.py cfg5 8 --noexit; done
done > gpurun_out/ablation.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_round_umma -c 1 -o gpurun_out/k5_w3 python tools/profile_round.py cfg5 8 > gpurun_out/ncu_k5.log 2>&1
