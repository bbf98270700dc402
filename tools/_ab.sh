cd $GRAFT_REPO_ROOT
# A/B of two library builds: per-launch durations (ncu) and the host-timed step
A=${1:-build/var/libbz_old.so}; B=${2:-paper_1603_06757_b200/libbz.so}
for lib in $A $B $A $B; do
echo $lib
BZ_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 5 python tools/round_stats.py cfg5 2>&1 | grep -E "duration" | awk '{print $2, $3}' | tr '\n' ' '; echo
BZ_LIB=$lib python tools/host_probe.py | grep flushed
done
