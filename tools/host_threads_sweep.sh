# one-shot call breakdown (C4, C2) at several host compile thread counts
cd "${GRAFT_REPO_ROOT:-.}"
for t in "8 4" "16 8" "12 6"; do
  set -- $t
  echo "TC_COMPILE_THREADS=$1 TC_TINY_THREADS=$2"
  TC_COMPILE_THREADS=$1 TC_TINY_THREADS=$2 python tools/e2e_breakdown.py c4 c2 2>&1 | grep -E '^c[0-9]'
done
