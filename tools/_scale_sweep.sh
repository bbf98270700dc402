cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do
for sc in 0.5 0.75 1 1.5 2 3; do
  echo "chunk scale $sc"; BZ_K5_CHUNK_SCALE=$sc python tools/shard_probe.py 8 | grep unsharded
done; done
