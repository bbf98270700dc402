cd $GRAFT_REPO_ROOT
for v in b2_e16_g1 b4_e16_g2 b4_e16_g4; do for g in 7 8; do echo "$v"; BZ_LIB=build/var/libbz_$v.so python tools/profile_round.py cfg5 $g --upper=20; done; done > gpurun_out/var.txt 2>&1
BZ_LIB=build/var/libbz_b4_e16_g2.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "mxf4q" 2>&1 | tail -1
