# k_tiny evidence (under gpurun): per-node clock trace of the heaviest group
# (block 0) of every tiny launch of one eager slice, and one --set full capture
# of C2's first tiny launch with source-level stall sampling
TC_TINY_TRACE=1 timeout 300 python tools/tiny_trace.py c2 > /dev/null 2> gpurun_out/tiny_trace_c2.txt
TC_TINY_TRACE=1 timeout 300 python tools/tiny_trace.py c3 > /dev/null 2> gpurun_out/tiny_trace_c3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tiny -c 1 \
  -o gpurun_out/r2b_c2_tiny python tools/one_slice.py c2 > gpurun_out/ncu_tiny_r2b.log 2>&1
