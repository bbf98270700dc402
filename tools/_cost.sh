cd $GRAFT_REPO_ROOT
# K5 level cost-model sweep (BZ_K5_COST = clocks per tile, per prefix step)
for c in "650,3500" "650,2500" "650,5000" "500,3500" "850,3500" "650,3500"; do
echo "cost $c"
BZ_K5_COST=$c ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 5 python tools/round_stats.py cfg5 2>&1 | grep -E "duration" | awk '{print $2, $3}' | tr '\n' ' '; echo
BZ_K5_COST=$c python tools/host_probe.py | grep "flushed step"
done
