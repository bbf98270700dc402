cd $GRAFT_REPO_ROOT
for lib in build/var/libbz_old.so paper_1603_06757_b200/libbz.so build/var/libbz_old.so paper_1603_06757_b200/libbz.so; do
echo $lib
BZ_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 5 python tools/round_stats.py cfg5 2>&1 | grep -E "duration" | awk '{print $2, $3}' | tr '\n' ' '; echo
done
