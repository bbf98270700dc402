cd $GRAFT_REPO_ROOT
for c in 880,1271 620,3000 620,600 700,5000; do for g in 7 8; do echo "$c"; BZ_K5_COST=$c python tools/profile_round.py cfg5 $g --upper=20; done; done > gpurun_out/cost.txt 2>&1
