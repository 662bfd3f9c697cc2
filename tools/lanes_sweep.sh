# C4 device + e2e at several slice-lane counts (TC_LANES), full bench lines
cd "${GRAFT_REPO_ROOT:-.}"
for l in 2 3 4 6 8; do
  TC_LANES=$l timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c2 > gpurun_out/s6_l$l.json 2>gpurun_out/s6_l$l.err
  python -c "import json; d=json.load(open('gpurun_out/s6_l$l.json')); print('lanes $l', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['e2e']['seconds_each'], d['device_peak_bytes'])" >> gpurun_out/s6_summary.txt 2>&1
done
