cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do for mg in 0 1; do
  echo "BZ_K5_MERGE=$mg"; BZ_K5_MERGE=$mg python tools/shard_probe.py 8 | grep "unsharded"
done; done
