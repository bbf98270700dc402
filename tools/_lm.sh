cd $GRAFT_REPO_ROOT
# chunk-size sweep: BZ_K5_LANE_MIN (small rounds) x BZ_K5_CHUNK_SCALE (all K5 rounds)
for cfg in "4096 1" "8192 1" "8192 1.5" "8192 2" "32768 1.5" "4096 1"; do
set -- $cfg
echo "lane_min $1 scale $2"
BZ_K5_LANE_MIN=$1 BZ_K5_CHUNK_SCALE=$2 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 5 python tools/round_stats.py cfg5 2>&1 | grep -E "duration" | awk '{print $2, $3}' | tr '\n' ' '; echo
BZ_K5_LANE_MIN=$1 BZ_K5_CHUNK_SCALE=$2 python tools/host_probe.py | grep "flushed step"
done
