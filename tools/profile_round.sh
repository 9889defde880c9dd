#!/bin/bash
# Profiling recipe for the committed evidence under profiles/ (run under gpurun).
#  1. launch list of the bench command (serialised, cold-cache: compare shares)
#  2. one ncu --set full capture of each kernel of a batched cfg2 step
set -x
mkdir -p gpurun_out
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline \
    > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
# tag:kernel-regex (the epoch-format merge kernels of the default key format)
for kk in trace_bundle:trace_bundle populate_depth:populate_depth dilate_rows:dilate_rows dilate_tiles:dilate_tiles \
          merge_shift:merge_epoch_kernel; do
  k=${kk%%:*}; re=${kk##*:}
  ncu --set full --clock-control none --import-source on -k regex:$re -s 4 -c 1 -o gpurun_out/${TAG}_$k \
      python tools/prof_frames.py cfg2x64 > gpurun_out/${TAG}_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:merge_sequence_epoch -s 2 -c 1 -o gpurun_out/${TAG}_merge_sequence \
    python tools/prof_frames.py seq64 > gpurun_out/${TAG}_merge_sequence.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:merge_epoch_tma -s 2 -c 1 -o gpurun_out/${TAG}_merge_tma \
    python tools/prof_frames.py odd8 > gpurun_out/${TAG}_merge_tma.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${TAG}_gpu.txt
