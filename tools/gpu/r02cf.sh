# throughput curve over the batch size (cfg2 and cfg1), current build
VXM_LIB_NAME=libvxm.so QT_CONFIGS="cfg2:1,cfg2:2,cfg2:4,cfg2:8,cfg2:12,cfg2:16,cfg2:24,cfg2:32,cfg2:64,cfg1:8,cfg1:16" timeout 600 python tools/quick_time.py 2>&1 | grep -v "^$" > gpurun_out/r02cf_curve.txt
cat gpurun_out/r02cf_curve.txt
