# round-2 final evidence (run under gpurun; outputs in gpurun_out/): every bench line,
# the reference arm, the ncu launch list of the default bench command and one
# --set full capture of the dominant per-slice stream kernel
set -x
bash tools/bench_all.sh
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/r2_c4_bench_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c2 > gpurun_out/r2_c4_bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 200 -c 2 \
  -o gpurun_out/r2b_c4_stream python tools/one_slice.py c4 --run-slices 2 > gpurun_out/ncu_full_r2b.log 2>&1
ls -la gpurun_out/ > gpurun_out/round_end_ls.txt
