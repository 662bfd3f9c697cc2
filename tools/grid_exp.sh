# stream grid multiplier experiment (mid-size launches, 2^10-2^11 chunks)
for m in 4 8 16; do
  TC_STREAM_GRID_MID=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/grid_c4_$m.json 2>/dev/null
  TC_STREAM_GRID_MID=$m timeout 300 python bench.py --config c5 --sample 128 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/grid_c5_$m.json 2>/dev/null
done
for m in 8 16 32; do
  TC_STREAM_GRID_MULT=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gridall_c4_$m.json 2>/dev/null
done
timeout 300 python tools/gemm_bench.py 10:10:12 10:13:8 6:14:5 13:13:13 > gpurun_out/gemm_bench.txt 2>&1
