cd ${GRAFT_REPO_ROOT:-.}
for ow in 6e8 1e8 1e7 1e5 0; do
  echo "BZ_OWN_WHOLE=$ow"
  BZ_OWN_WHOLE=$ow python tools/shard_probe.py 8 | grep "batch per shard"
  BZ_OWN_WHOLE=$ow python tools/shard_probe.py 4 | grep "batch per shard"
done
