cd $GRAFT_REPO_ROOT
for lib in paper_1603_06757_b200/libbz.so build/var/libbz_f32.so; do
  for g in 11 12; do BZ_LIB=$lib python tools/profile_s6.py C1 $g; BZ_LIB=$lib python tools/profile_s6.py C1 $g; done
done
BZ_LIB=build/var/libbz_f32.so timeout 600 python -m pytest tests/test_gpu_section6.py -x -q 2>&1 | tail -2
