cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do
for c in 650,3500 650,8000 650,12000 650,20000 650,40000; do
  echo "cost $c"; BZ_K5_COST=$c python tools/shard_probe.py 8 | grep unsharded
done; done
