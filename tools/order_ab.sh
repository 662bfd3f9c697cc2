# slice order A/B (TC_SLICE_ORDER=0: lexicographic blocks of 2) + the GPU suite
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/s18_tests.log 2>&1; echo tests_exit $? >> $O/s18_tests.log
for v in 1 0; do TC_SLICE_ORDER=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c2 > $O/s18_c4_o$v.json 2>$O/s18_c4_o$v.err; done
for v in 1 0; do TC_SLICE_ORDER=$v timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-c2 > $O/s18_c5_o$v.json 2>$O/s18_c5_o$v.err; done
