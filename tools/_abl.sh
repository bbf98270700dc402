cd $GRAFT_REPO_ROOT
for g in 5 6 7 8; do echo "g=$g"; BZ_K4_DEBUG=32 BZ_K4_CTRACE=gpurun_out/ct$g.bin python tools/profile_round.py cfg5 $g --upper=25 --engine=mxf4q; python tools/chunk_times.py gpurun_out/ct$g.bin; done > gpurun_out/ct.txt 2>&1
