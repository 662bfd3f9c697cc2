cd "${GRAFT_REPO_ROOT:-.}"
for env in "TC_BLOCK=1" "TC_BLOCK=0" "TC_LANES=1" "TC_OVERLAP_BUILD=0"; do
  env $env python tools/block_debug.py c1b_s3 0 8
  env $env python tools/block_debug.py c1b_s3 2 6
  env $env python tools/block_debug.py c1b_s3 1 6
done
