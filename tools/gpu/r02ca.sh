# K1 face hint from the slot's previous frame (libvxm) vs HEAD (per-tile switch only) vs 88b145a (serial)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_trajectory.py tests/test_gpu_sequence.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r02ca_tests.txt
for rep in 1 2; do for lib in libvxm_pub.so libvxm_head.so libvxm.so; do
  echo "== $lib $(VXM_LIB_NAME=$lib timeout 300 python tools/probes/traj_probe.py 2>&1 | tail -1)"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:64,cfg2:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02ca_ab.txt 2>&1
cat gpurun_out/r02ca_tests.txt; grep -v stages gpurun_out/r02ca_ab.txt
