cd $GRAFT_REPO_ROOT
for v in b2_e16 b3_e16 b2_e8 b3_e8 b3_e12; do for e in mxf4q; do
  echo "$v $e"; BZ_LIB=build/var/libbz_$v.so python tools/profile_round.py cfg5 8 --engine=$e --upper=18;  BZ_LIB=build/var/libbz_$v.so python tools/profile_round.py cfg5 8 --engine=$e --upper=18
done; done > gpurun_out/var.txt 2>&1
