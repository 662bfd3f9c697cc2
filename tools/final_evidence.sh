# round-2 final evidence (run under gpurun; outputs in gpurun_out/final_*): every bench
# line (W >= 3), the reference arm, the ncu launch list of the default bench command and
# one --set full capture of the dominant per-slice stream-pair kernel
cd "${GRAFT_REPO_ROOT:-.}"
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $O/final_smi.txt
timeout 600 python bench.py --steps 10 --warmup 3 > $O/final_bench_c4_n1.json 2> $O/final_bench_c4_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/final_bench_c4_reference.json 2> $O/final_bench_c4_reference.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > $O/final_bench_c2_n1.json 2> $O/final_bench_c2_n1.err
timeout 600 python bench.py --config c1a --steps 10 --warmup 3 > $O/final_bench_c1a_n1.json 2> $O/final_bench_c1a_n1.err
timeout 600 python bench.py --config c1b --steps 10 --warmup 3 > $O/final_bench_c1b_n1.json 2> $O/final_bench_c1b_n1.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 > $O/final_bench_c3_n1.json 2> $O/final_bench_c3_n1.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > $O/final_bench_c5_n1.json 2> $O/final_bench_c5_n1.err
timeout 600 python bench.py --config c4_full --steps 5 --warmup 3 --no-cpu-baseline > $O/final_bench_c4_full_n1.json 2> $O/final_bench_c4_full_n1.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file $O/final_c4_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c2 > $O/final_c4_bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_pair -s 200 -c 1 \
  -o $O/final_c4_pair python tools/one_slice.py c4 --run-slices 2 > $O/final_ncu_full.log 2>&1
ls -la $O/ > $O/final_ls.txt
