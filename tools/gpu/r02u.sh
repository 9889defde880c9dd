# dedup variants: RED count, MIO/issue metrics, duration for cfg1 and cfg2 batches
M=gpu__time_duration.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,lts__t_requests_op_red.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__average_warp_latency_issue_stalled_mio_throttle,smsp__average_warp_latency_issue_stalled_short_scoreboard,lts__t_sectors_op_red.sum
for cfg in cfg2x64 cfg1x64; do
for lib in libvxm_cur.so libvxm_shfl.so; do
  echo "== $cfg $lib"
  VXM_LIB_NAME=$lib ncu --metrics $M --clock-control none -k regex:trace_bundle -s 4 -c 1 --csv python tools/prof_frames.py $cfg 2>/dev/null | grep -v "^==" | tail -n +2 | awk -F'","' '{print $(NF-2), $NF}'
done
done > gpurun_out/r02u_dedup.txt 2>&1
cat gpurun_out/r02u_dedup.txt
