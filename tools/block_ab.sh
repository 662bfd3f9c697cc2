# slice blocks A/B (TC_BLOCK=0: block tier per slice) + the GPU suite
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
for v in 1 0; do for c in c4 c1b; do TC_BLOCK=$v timeout 300 python tools/diag_pass.py $c | sed "s/^/block$v /"; done; done > $O/s11_block.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/s11_tests.log 2>&1; echo tests_exit $? >> $O/s11_tests.log
for v in 1 0; do TC_BLOCK=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c2 > $O/s11_c4_b$v.json 2>$O/s11_c4_b$v.err; done
for v in 1 0; do TC_BLOCK=$v timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-c2 > $O/s11_c5_b$v.json 2>$O/s11_c5_b$v.err; done
