# round-2 ncu evidence (run under gpurun; outputs in gpurun_out/)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in 1 2; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_c4_launches_$k.csv \
    python tools/one_slice.py c4 --run-slices $k > gpurun_out/ncu_$k.log 2>&1
done
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_c3_launches_1.csv \
  python tools/one_slice.py c3 --run-slices 1 > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 40 -c 1 \
  -o gpurun_out/r2_c4_stream_pro python tools/one_slice.py c4 > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 250 -c 2 \
  -o gpurun_out/r2_c4_stream_var python tools/one_slice.py c4 --run-slices 2 > gpurun_out/ncu_full2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 20 -c 3 \
  -o gpurun_out/r2_c3_gemm python tools/one_slice.py c3 > gpurun_out/ncu_full3.log 2>&1
ls -la gpurun_out/ > gpurun_out/ncu_ls.txt
