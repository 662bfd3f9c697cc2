# round-2b --set full capture of the largest per-slice stream-pair launch of one C4
# slice pass (picked from the launch list of the same command)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2b_c4_launches_1.csv \
  python tools/one_slice.py c4 --run-slices 1 > gpurun_out/ncu_r2b_list.log 2>&1
N=$(python tools/ncu_pick.py gpurun_out/r2b_c4_launches_1.csv k_stream_pair --first 190)
echo "pair launch $N" > gpurun_out/ncu_r2b_pick.txt
timeout 900 ncu --set full --clock-control none --import-source on --launch-skip $N --launch-count 1 \
  -o gpurun_out/r2b_c4_pair python tools/one_slice.py c4 --run-slices 1 > gpurun_out/ncu_r2b_full.log 2>&1
