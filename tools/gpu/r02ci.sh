# K3 tail-fast in the one-warp kernel only: parity, fuzz, lone/batch timing vs HEAD
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sequence.py tests/test_gpu_trajectory.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r02ci_tests.txt
timeout 400 python tools/fuzz_parity.py 240 701 2>&1 | tail -1 >> gpurun_out/r02ci_tests.txt
for rep in 1 2; do for lib in libvxm_head.so libvxm.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:1,cfg1:1,cfg3:1,cfg2:2,cfg2:4,cfg2:64" timeout 600 python tools/quick_time.py 2>&1 | grep graph
done; done > gpurun_out/r02ci_ab.txt 2>&1
cat gpurun_out/r02ci_tests.txt gpurun_out/r02ci_ab.txt
