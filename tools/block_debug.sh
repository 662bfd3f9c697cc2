# per-slice bits under the slice order / block tier / plain per-slice execution
cd "${GRAFT_REPO_ROOT:-.}"
for env in "TC_BLOCK=1" "TC_SLICE_ORDER=0" "TC_BLOCK=0" "TC_LANES=1"; do
  for r in "0 256" "32 64" "1 20" "8 40"; do env $env python tools/block_debug.py c4 $r; done
  for r in "3584 4096" "3584 3600" "0 512"; do env $env python tools/block_debug.py c5 $r; done
done
