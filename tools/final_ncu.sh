# --set full capture of the largest per-slice stream-pair launch of one C4 slice pass
# (picked from the launch list of the same command), final code of round 2
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/final_c4_slice_launches.csv \
  python tools/one_slice.py c4 --run-slices 1 > $O/final_ncu_list.log 2>&1
N=$(python tools/ncu_pick.py $O/final_c4_slice_launches.csv k_stream_pair --first 190)
echo "pair launch $N" > $O/final_ncu_pick.txt
timeout 900 ncu --set full --clock-control none --import-source on --launch-skip $N --launch-count 1 \
  -o $O/final_c4_pair python tools/one_slice.py c4 --run-slices 1 > $O/final_ncu_full.log 2>&1
