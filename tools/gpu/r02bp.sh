# chain merge: 128-thread blocks, U=8 at minB 4 (A/B vs HEAD)
VXM_LIB_NAME=libvxm_t128.so timeout 1200 python -m pytest tests/test_gpu_sequence.py tests/test_gpu_trajectory.py tests/test_gpu_keys.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r02bp_tests.txt
for rep in 1 2; do for lib in libvxm_head.so libvxm_t128.so libvxm_m4u8.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:1:64,cfg2:1:64,cfg3:1:16,cfg1:4:16" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02bp_ab.txt 2>&1
cat gpurun_out/r02bp_tests.txt gpurun_out/r02bp_ab.txt
