# K1 face hint threshold: 50% (h50), 75% (libvxm), 90% (h90) of warps vs HEAD (no hint)
true
for rep in 1 2; do for lib in libvxm_head.so libvxm_h50.so libvxm.so libvxm_h90.so; do
  echo "== $lib $(VXM_LIB_NAME=$lib timeout 300 python tools/probes/traj_probe.py 2>&1 | tail -1)"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:64,cfg2:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02cb_ab.txt 2>&1
cat gpurun_out/r02cb_tests.txt; grep -v stages gpurun_out/r02cb_ab.txt
