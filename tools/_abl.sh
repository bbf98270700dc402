cd $GRAFT_REPO_ROOT
for v in e16_g1 e16_g2 e24_g2; do for g in 7 8; do echo "$v"; BZ_LIB=build/var/libbz_$v.so python tools/profile_round.py cfg5 $g --upper=20; done; done > gpurun_out/var.txt 2>&1
for v in e16_g2 e24_g2; do BZ_LIB=build/var/libbz_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "mxf4q or cfg5 or weight_range" 2>&1 | tail -1; done
