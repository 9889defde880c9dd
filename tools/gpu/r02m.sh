set -x
ncu --set full --clock-control none --import-source on -k regex:trace_bundle -s 4 -c 1 -o gpurun_out/r02m_trace_bundle python tools/prof_frames.py cfg2x64 > gpurun_out/r02m_tb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:merge_epoch_kernel -s 4 -c 1 -o gpurun_out/r02m_merge python tools/prof_frames.py cfg2x64 > gpurun_out/r02m_mg.log 2>&1
ls -la gpurun_out/
