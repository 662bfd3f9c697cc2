# every bench line of the round (outputs in gpurun_out/)
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_c4_n1.json 2> gpurun_out/r2_bench_c4_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_c4_reference.json 2> gpurun_out/r2_bench_c4_reference.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/r2_bench_c2_n1.json 2> gpurun_out/r2_bench_c2_n1.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 2 > gpurun_out/r2_bench_c3_n1.json 2> gpurun_out/r2_bench_c3_n1.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/r2_bench_c5_n1.json 2> gpurun_out/r2_bench_c5_n1.err
timeout 600 python bench.py --config c1b --steps 10 --warmup 3 > gpurun_out/r2_bench_c1b_n1.json 2> gpurun_out/r2_bench_c1b_n1.err
timeout 600 python bench.py --config c4_full --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_c4_full_n1.json 2> gpurun_out/r2_bench_c4_full_n1.err
