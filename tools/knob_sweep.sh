cd "${GRAFT_REPO_ROOT:-.}"
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c2 --e2e-steps 1 > gpurun_out/s4_$tag.json 2>gpurun_out/s4_$tag.err; python -c "import json; d=json.load(open('gpurun_out/s4_$tag.json')); print('$tag', round(d['ms_per_step'],2), d['parity']['max_rel_err'])" >> gpurun_out/s4_summary.txt 2>&1; }
run base
run p11 TC_STREAM_PERSIST=11
run p10 TC_STREAM_PERSIST=10
run p9 TC_STREAM_PERSIST=9
run mid8 TC_STREAM_GRID_MID=8
run mid2 TC_STREAM_GRID_MID=2
run p10l6 TC_STREAM_PERSIST=10 TC_LANES=6
run l6 TC_LANES=6
