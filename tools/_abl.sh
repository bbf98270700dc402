cd $GRAFT_REPO_ROOT
for e in auto mxf4q popc; do for g in 4 5 6 7 8; do echo "$e"; python tools/profile_round.py cfg5 $g --upper=25 --engine=$e; done; done 2>&1 > gpurun_out/warm.txt
