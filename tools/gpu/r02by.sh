# K1 near-integer floor placement: in-loop batch 4 (libvxm) / 2 (nb2), after the loop batch 4 (np4) / 2 (np2), vs 88b145a (pub)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectory.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r02by_tests.txt
for rep in 1 2; do for lib in libvxm_pub.so libvxm.so libvxm_nb2.so libvxm_np4.so libvxm_np2.so; do
  echo "== $lib $(VXM_LIB_NAME=$lib timeout 300 python tools/probes/traj_probe.py 2>&1 | tail -1)"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:64,cfg2:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02by_ab.txt 2>&1
cat gpurun_out/r02by_tests.txt; grep -v stages gpurun_out/r02by_ab.txt
