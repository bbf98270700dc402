cd ${GRAFT_REPO_ROOT:-.}
for c in 727,1271 727,3000 727,6000 727,12000 727,24000; do
  echo "cost $c"; for g in 10 12; do BZ_K5_COST=$c python tools/profile_s6.py C1 $g | tail -1; done
done
echo "merge off"; BZ_K5_MERGE=0 python tools/profile_s6.py C1 12 | tail -1
